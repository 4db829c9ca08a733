"""Summarise a GPU round's ncu outputs (gpurun_out/) into profiles/ (tracked).

    python tools/summarize_profiles.py r1 [--workload bf16_4096]

Writes profiles/<tag>_launches.md (per-kernel share of the launch list),
profiles/<tag>_ncu_<kernel>.md (key metrics of the ncu --set full capture) and
profiles/traffic_<workload>.json (DRAM bytes per launch of the captured config, read by bench.py).
"""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "launch__shared_mem_per_block_dynamic", "sm__cycles_elapsed.avg.per_second",
    "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
]


def launches(tag):
    path = os.path.join(OUT, f"launches_{tag}.csv")
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rd = csv.DictReader(lines)
    for r in rd:
        if r.get("Metric Name") == "gpu__time_duration.sum":
            v = float(r["Metric Value"].replace(",", ""))
            unit = r.get("Metric Unit", "")
            scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}.get(unit, 1.0)
            rows.append((r["Kernel Name"], v * scale))
    by = collections.defaultdict(lambda: [0, 0.0])
    for k, t in rows:
        short = k.split("(")[0][:90]
        by[short][0] += 1
        by[short][1] += t
    tot = sum(v[1] for v in by.values())
    lines = [f"# Launch list {tag} (ncu --metrics gpu__time_duration.sum --clock-control none)", "",
             f"Command: `python bench.py --steps 5 --warmup 3 --no-cpu-baseline` (tuning pass + timed steps).",
             f"{len(rows)} launches, {tot / 1e3:.2f} ms total device time (cold-cache, serialised).", "",
             "| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k, (n, t) in sorted(by.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{k}` | {n} | {t:.1f} | {100 * t / tot:.1f} % |")
    with open(os.path.join(PROF, f"{tag}_launches.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    return by


def ncu_metrics(tag):
    rep = os.path.join(OUT, f"prof_{tag}.ncu-rep")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(raw.splitlines()))
    h, u, v = r[0], r[1], r[2]
    got = {}
    for i, n in enumerate(h):
        if n in KEYS:
            got[n] = (v[i], u[i])
    name = v[h.index("Kernel Name")] if "Kernel Name" in h else "k_umma"
    return name, got


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
    workload = "bf16_4096"
    if "--workload" in sys.argv:
        workload = sys.argv[sys.argv.index("--workload") + 1]
    os.makedirs(PROF, exist_ok=True)
    launches(tag)
    name, m = ncu_metrics(tag)
    bench = json.load(open(os.path.join(OUT, f"bench_{tag}.json")))
    cfg = bench["config"]["best_config"]
    dram = None
    if "dram__bytes_read.sum" in m and "dram__bytes_write.sum" in m:
        def to_bytes(val, unit):
            x = float(val.replace(",", ""))
            return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        dram = to_bytes(*m["dram__bytes_read.sum"]) + to_bytes(*m["dram__bytes_write.sum"])
    lines = [f"# ncu --set full: {name.split('(')[0]} ({tag})", "",
             f"Config {json.dumps(cfg)} of workload {workload}; captured with "
             "`ncu --set full --clock-control none --import-source on -k regex:k_umma -s 3 -c 1` "
             "(one launch after 3 skipped, L2 flushed before it).", "",
             "| metric | value | unit |", "|---|---|---|"]
    for k in KEYS:
        if k in m:
            lines.append(f"| `{k}` | {m[k][0]} | {m[k][1]} |")
    M, N, K = bench["config"]["M_per_rank"], bench["config"]["N"], bench["config"]["K"]
    alg_in = (M * K + K * N) * (2 if bench["dtype"] == "bf16" else 4)
    alg = alg_in + M * N * 4
    if dram:
        lines += ["", f"DRAM traffic per launch {dram / 1e6:.1f} MB vs compulsory {alg / 1e6:.1f} MB "
                  f"(A + B in, C out): ratio {dram / alg:.2f}.  C write-back that is still in L2 when the kernel "
                  "ends is not counted by the kernel's DRAM counters."]
    with open(os.path.join(PROF, f"{tag}_ncu_k_umma.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    clk = m.get("sm__cycles_elapsed.avg.per_second")
    ten = m.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed")
    extra = {}
    if clk:
        g = float(clk[0].replace(",", "")) * {"Ghz": 1.0, "Mhz": 1e-3, "hz": 1e-9}.get(clk[1], 1.0)
        extra = {"sm_clock_ghz_ncu": g, "tensor_active_pct_ncu": float(ten[0]) if ten else None,
                 "clock_source": f"sm__cycles_elapsed.avg.per_second / sm__pipe_tensor_cycles_active of the {tag} "
                                 f"--set full capture (profiles/{tag}_ncu_k_umma.md)"}
    merge_traffic(tag, workload, [cfg["m"], cfg["k"], cfg["n"]], extra)
    print("wrote", tag)


def merge_traffic(tag, workload, cfg, extra=None):
    """Update the bench config's entry of profiles/traffic_<workload>.json (the table bench.py's
    roofline.traffic reads) from gpurun_out/traffic_<tag>.csv (ncu --metrics dram bytes of one
    launch of that config under the current build)."""
    path = os.path.join(OUT, f"traffic_{tag}.csv")
    if not os.path.exists(path):
        return
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    vals = {}
    for r in csv.DictReader(lines):
        x = float(r["Metric Value"].replace(",", ""))
        x *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6}.get(
            r.get("Metric Unit", ""), 1)
        vals[r["Metric Name"]] = x
    entry = {"config": cfg, "dram_bytes_per_launch": vals.get("dram__bytes_read.sum", 0) + vals.get("dram__bytes_write.sum", 0),
             "dram_read": vals.get("dram__bytes_read.sum"), "dram_write": vals.get("dram__bytes_write.sum"),
             "lts_bytes": vals.get("lts__t_bytes.sum"), "ncu_duration_ns": vals.get("gpu__time_duration.sum"),
             "captured": f"{tag} (tools/gpu_{tag}_final.sh, current split policy)"}
    entry.update(extra or {})
    tp = os.path.join(PROF, f"traffic_{workload}.json")
    table = json.load(open(tp)) if os.path.exists(tp) else {"workload": workload, "configs": []}
    table.setdefault("configs", [])
    table["configs"] = [e for e in table["configs"] if e.get("config") != cfg] + [entry]
    with open(tp, "w") as f:
        json.dump(table, f, indent=1)


if __name__ == "__main__":
    main()

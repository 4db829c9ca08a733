"""Render one `ncu --set full` report into a markdown summary for profiles/ (run on the CPU box).

    python tools/ncu_summary.py gpurun_out/prof_r10_f32_4096.ncu-rep "title" [--flops F] [--bytes B] > profiles/x.md

Prints: duration and clock, pipe utilisation (tensor, FMA), DRAM / L2 traffic against the given
algorithmic flops / bytes, occupancy, shared-memory wavefronts and bank conflicts, the warp-stall
breakdown (per issued instruction) and the SASS opcodes that hold the most stall samples.
"""
import argparse
import collections
import csv
import io
import subprocess

METRICS = [
    ("gpu__time_duration.sum", "kernel duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("launch__grid_size", "grid (CTAs)"),
    ("launch__block_size", "block (threads)"),
    ("launch__cluster_size", "cluster size"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem / CTA"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active (of max)"),
    ("sm__cycles_active.avg", "SM active cycles (avg)"),
    ("gpc__cycles_elapsed.avg", "elapsed cycles"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active (of active cycles)"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active (of elapsed)"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe active (of active cycles)"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_elapsed", "FMA pipe active (of elapsed)"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA-pipe instructions issued (of peak)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput (of peak)"),
    ("lts__t_bytes.sum", "L2 traffic (lts__t_bytes)"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput (of peak)"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shared-memory wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "shared-memory bank conflicts"),
]


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True, check=True).stdout


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("title")
    ap.add_argument("--flops", type=float, default=None, help="algorithmic flops per launch")
    ap.add_argument("--bytes", type=float, default=None, help="compulsory DRAM bytes per launch")
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    raw = list(csv.reader(io.StringIO(ncu("-i", a.rep, "--page", "raw", "--csv"))))
    hdr, units, vals = raw[0], raw[1], raw[2]
    get = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
    name = get.get("Kernel Name", ("?", ""))[0]
    print(f"# {a.title}\n")
    print(f"Source: `{a.rep.split('/')[-1]}` (ncu `--set full --clock-control none`, one launch after an L2 flush; "
          f"ncu serialises and cold-starts each replay, so compare shares and counters, not absolute speed).\n")
    print(f"Kernel: `{name[:160]}`\n")
    if a.note:
        print(a.note + "\n")
    print("| metric | value |\n|---|---|")
    for key, label in METRICS:
        if key in get and get[key][0] not in ("", "n/a"):
            v, u = get[key]
            print(f"| {label} (`{key}`) | {v} {u} |")
    dur = get.get("gpu__time_duration.sum")
    if dur:
        t = float(dur[0].replace(",", "")) * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3,
                                              "nsecond": 1e-9}.get(dur[1], 1e-6)
        if a.flops:
            print(f"| achieved (algorithmic flops / duration) | {a.flops / t / 1e12:.1f} TFLOP/s |")
        if a.bytes:
            rd = float(get["dram__bytes_read.sum"][0].replace(",", "")) * (1e6 if get["dram__bytes_read.sum"][1] == "Mbyte" else (1e3 if get["dram__bytes_read.sum"][1] == "Kbyte" else (1e9 if get["dram__bytes_read.sum"][1] == "Gbyte" else 1)))
            wr = float(get["dram__bytes_write.sum"][0].replace(",", "")) * (1e6 if get["dram__bytes_write.sum"][1] == "Mbyte" else (1e3 if get["dram__bytes_write.sum"][1] == "Kbyte" else (1e9 if get["dram__bytes_write.sum"][1] == "Gbyte" else 1)))
            print(f"| DRAM traffic / compulsory bytes | {(rd + wr) / a.bytes:.2f} ({(rd + wr) / 1e6:.1f} MB vs {a.bytes / 1e6:.1f} MB) |")
    print("\n## Warp stalls (warps stalled per issued instruction)\n")
    print("| reason | per issue |\n|---|---|")
    st = []
    for h in hdr:
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                v = float(get[h][0])
            except ValueError:
                continue
            if v >= 0.01:
                st.append((v, h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
    for v, n in sorted(st, reverse=True):
        print(f"| {n} | {v:.3f} |")
    src = list(csv.reader(io.StringIO(ncu("-i", a.rep, "--page", "source", "--csv", "--print-source", "sass"))))
    shdr, rows = src[1], src[2:]
    i_src, i_s = shdr.index("Source"), shdr.index("Warp Stall Sampling (All Samples)")
    ops = collections.Counter()
    tot = 0
    for r in rows:
        n = int(r[i_s] or 0)
        tot += n
        toks = r[i_src].strip().split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        ops[op.split(".")[0]] += n
    print(f"\n## Stall samples by SASS opcode ({tot} samples)\n")
    print("| opcode | share |\n|---|---|")
    for op, n in ops.most_common(10):
        print(f"| {op} | {100.0 * n / max(tot, 1):.1f} % |")


if __name__ == "__main__":
    main()

"""Debug timeline of the persistent tcgen05 kernel (TT_UMMA_TRACE, DESIGN.md §6 tail split).

Runs one config a few times with the item trace on and prints, per cluster, each item's tile,
k-range, order and timestamps relative to the kernel's earliest MMA start (us)."""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=4096)
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--k", type=int, default=4096)
    ap.add_argument("--family", default="bf16")
    ap.add_argument("--config", required=True)
    ap.add_argument("--out", default="gpurun_out/umma_trace.bin")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--mhz", type=float, default=1965.0, help="SM clock for cycles -> us")
    ap.add_argument("--flush", action="store_true", help="256 MiB memset before every launch (bench protocol)")
    a = ap.parse_args()
    if os.path.exists(a.out):
        os.remove(a.out)
    os.environ["TT_UMMA_TRACE"] = a.out
    # the trace instrumentation exists only in the trace build of the library
    lib = os.path.join(ROOT, "build", "variants", "trace", "libtiletune.so")
    if not os.path.exists(lib):
        sys.path.insert(0, ROOT)
        from paper_1909_10616_b200 import build
        lib = build.build_variant("trace", ["TT_UMMA_TRACE_BUILD"])
    os.environ.setdefault("TT_LIB_PATH", lib)
    import torch
    from paper_1909_10616_b200 import tiletune as tt
    fam = {"bf16": tt.FAM_BF16_UMMA, "tf32": tt.FAM_TF32_UMMA}[a.family]
    cfg = json.loads(a.config)
    s = (tuple(cfg["m"]), tuple(cfg["k"]), tuple(cfg["n"]))
    dt = torch.bfloat16 if a.family == "bf16" else torch.float32
    A = torch.randn(a.m, a.k, device="cuda").to(dt)
    B = torch.randn(a.k, a.n, device="cuda").to(dt)
    C = torch.empty(a.m, a.n, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda") if a.flush else None
    for r in range(a.reps):
        if flush is not None:
            flush.fill_(r & 0xFF)
            torch.cuda.synchronize()
        tt.gemm(A, B, C, fam, s)
    torch.cuda.synchronize()
    raw = np.fromfile(a.out, dtype=np.uint64)
    pos = 0
    rep = 0
    while pos < raw.size:
        ncl, nit, dp, sk = (int(x) for x in raw[pos:pos + 4])
        pos += 4
        tr = raw[pos:pos + ncl * nit * 8].reshape(ncl, nit, 8).astype(np.int64)
        pos += ncl * nit * 8
        rep += 1
        if rep < a.reps:
            continue
        valid = tr[:, :, 2] > 0
        t0 = tr[:, :, 2][valid].min()
        end = tr[:, :, 6][valid].max()
        entry = tr[:, 0, 7]
        teardown = tr[:, 1, 7]
        print(f"clusters {ncl} dp_tiles {dp} sk_tiles {sk} kernel span {(end - t0) / 1e3:.2f} us; "
              f"entry {(entry.min() - t0) / 1e3:.2f} .. {(entry.max() - t0) / 1e3:.2f} us, "
              f"teardown passed {(teardown.max() - t0) / 1e3:.2f} us (relative to the first MMA)")
        for k, what in ((2, "barriers initialised"), (3, "TMEM allocated"), (4, "prologue barrier passed"),
                        (5, "MMA role set up"), (6, "first TMA issued"),
                        (7, "first stage landed")):
            v = tr[:, k, 7]
            v = v[v > 0]
            if v.size:
                print(f"  {what}: {(v.min() - t0) / 1e3:.2f} .. {(v.max() - t0) / 1e3:.2f} us")
        names = ["barriers init", "TMEM alloc", "prologue barrier", "first TMA issue", "first stage landed",
                 "item 0 last MMA commit", "item 0 epilogue done", "teardown"]
        cyc = tr[:, 8:16, 7]
        print("  per-CTA cycles since entry (median over clusters; us at %.0f MHz):" % a.mhz)
        for i, nm in enumerate(names):
            v = cyc[:, i]
            v = v[v > 0]
            if v.size:
                print(f"    {nm:24s} {int(np.median(v)):7d} cyc  {np.median(v) / a.mhz:6.2f} us  "
                      f"(min {v.min() / a.mhz:.2f} max {v.max() / a.mhz:.2f})")
        ends = []
        for c in range(ncl):
            items = []
            for i in range(nit):
                if tr[c, i, 2] == 0:
                    break
                tile, w, ms, me, ea, ef, ed, _ = tr[c, i]
                kb0, kb1, order = w & 0xFFFF, (w >> 16) & 0xFFFF, w >> 32
                items.append(f"t{tile}[{kb0},{kb1})o{order} mma {(ms - t0) / 1e3:.1f}-{(me - t0) / 1e3:.1f} "
                             f"epi {(ea - t0) / 1e3:.1f}/{(ef - t0) / 1e3:.1f}/{(ed - t0) / 1e3:.1f}")
            ends.append((tr[c, :, 6].max() - t0) / 1e3)
            if c < 12 or c % 10 == 0:
                print(f"c{c:3d}: " + " | ".join(items))
        ends = np.array(ends)
        print(f"cluster end us: min {ends.min():.1f} median {np.median(ends):.1f} max {ends.max():.1f}")


if __name__ == "__main__":
    main()

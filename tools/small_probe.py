"""Cold- and warm-L2 timing of tcgen05 configs on one problem (profiling aid, not a test).

    python tools/small_probe.py M N K fam [--all] [--split 0|1|2] [--reps 20] [--cfg JSON ...]

Cold = a 256 MiB memset before every launch (bench.py's protocol), events around the launch only.
Warm = back-to-back launches.  Prints one JSON line per config.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("M", type=int)
    ap.add_argument("N", type=int)
    ap.add_argument("K", type=int)
    ap.add_argument("fam", type=int)
    ap.add_argument("--all", action="store_true", help="every feasible config")
    ap.add_argument("--cfg", action="append", default=[])
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--top", type=int, default=0, help="print only the best N (cold)")
    args = ap.parse_args()
    import torch

    from paper_1909_10616_b200 import tiletune as tt
    dev = torch.device("cuda:0")
    M, N, K, fam = args.M, args.N, args.K, args.fam
    sp = tt.make_space(M, N, K, family=fam)
    dt = torch.bfloat16 if fam == 3 else torch.float32
    A = torch.empty(M, K, device=dev, dtype=dt)
    B = torch.empty(K, N, device=dev, dtype=dt)
    C = torch.empty(M, N, device=dev)
    tt.fill_uniform(A, 1)
    tt.fill_uniform(B, 2)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    cfgs = [tuple(tuple(v) for v in json.loads(c)) for c in args.cfg]
    if args.all:
        cfgs += tt.enumerate_feasible(sp)[0]
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.reps + 2)]
    out = []
    for cfg in cfgs:
        info = tt.binding(sp, cfg)
        for _ in range(3):
            tt.gemm(A, B, C, fam, cfg)
        torch.cuda.synchronize()
        cold = []
        for r in range(args.reps):
            flush.fill_(r & 0xFF)
            ev[0].record()
            tt.gemm(A, B, C, fam, cfg)
            ev[1].record()
            torch.cuda.synchronize()
            cold.append(ev[0].elapsed_time(ev[1]) * 1e3)
        ev[0].record()
        for r in range(args.reps):
            tt.gemm(A, B, C, fam, cfg)
        ev[1].record()
        torch.cuda.synchronize()
        warm = ev[0].elapsed_time(ev[1]) * 1e3 / args.reps
        cold.sort()
        med = cold[len(cold) // 2]
        rec = {"cfg": cfg, "cold_us": med, "cold_min_us": cold[0], "warm_us": warm,
               "cold_tflops": 2 * M * N * K / (med * 1e-6) / 1e12, "grid": info.grid_x, "cluster": info.cluster_x,
               "tile": [info.tile_m, info.tile_n, info.tile_k], "stages": info.stages, "split": info.split_tiles,
               "split_workers": info.split_workers}
        out.append(rec)
        if not args.top:
            print(json.dumps(rec), flush=True)
    if args.top:
        for rec in sorted(out, key=lambda r: r["cold_us"])[:args.top]:
            print(json.dumps(rec))


if __name__ == "__main__":
    main()

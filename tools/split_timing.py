"""Tail-split A/B timing: one config, isolated launches (sync between) vs
back-to-back launches, CUDA events; run once with TT_TAIL_SPLIT=1 and once with 0."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=4096)
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--k", type=int, default=4096)
    ap.add_argument("--family", default="bf16")
    ap.add_argument("--config", required=True)
    a = ap.parse_args()
    import torch
    from paper_1909_10616_b200 import tiletune as tt
    fam = {"bf16": tt.FAM_BF16_UMMA, "tf32": tt.FAM_TF32_UMMA}[a.family]
    cfg = json.loads(a.config)
    s = (tuple(cfg["m"]), tuple(cfg["k"]), tuple(cfg["n"]))
    dt = torch.bfloat16 if a.family == "bf16" else torch.float32
    A = torch.randn(a.m, a.k, device="cuda").to(dt)
    B = torch.randn(a.k, a.n, device="cuda").to(dt)
    C = torch.empty(a.m, a.n, device="cuda")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for _ in range(5):
        tt.gemm(A, B, C, fam, s)
    torch.cuda.synchronize()
    iso = []
    for _ in range(20):
        ev[0].record()
        tt.gemm(A, B, C, fam, s)
        ev[1].record()
        torch.cuda.synchronize()
        iso.append(ev[0].elapsed_time(ev[1]) * 1e3)
        time.sleep(0.002)
    iso.sort()
    b2b = {}
    for n in (5, 50, 500):
        ev[0].record()
        for _ in range(n):
            tt.gemm(A, B, C, fam, s)
        ev[1].record()
        torch.cuda.synchronize()
        b2b[n] = ev[0].elapsed_time(ev[1]) * 1e3 / n
    # host launch cost: enqueue time of 200 launches behind a long-running kernel
    torch.cuda._sleep(200_000_000)
    t0 = time.perf_counter()
    for _ in range(200):
        tt.gemm(A, B, C, fam, s)
    host_us = (time.perf_counter() - t0) / 200 * 1e6
    torch.cuda.synchronize()
    info = tt.binding(tt.make_space(a.m, a.n, a.k, family=fam), s)
    print(json.dumps({"split": os.environ.get("TT_TAIL_SPLIT", "1"), "config": cfg, "split_tiles": info.split_tiles,
                      "iso_us_median": iso[len(iso) // 2], "iso_us_min": iso[0], "b2b_us": b2b,
                      "host_us_per_launch": host_us}))


if __name__ == "__main__":
    main()

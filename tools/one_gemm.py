"""Launch one config a few times (each after an L2-flush memset) -- the command ncu profiles.

    python tools/one_gemm.py M N K fam '[[m..],[k..],[n..]]' [--n 3] [--layout nn|tn]
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
    ap.add_argument("cfg")
    ap.add_argument("--n", type=int, default=3)
    ap.add_argument("--layout", default="nn")
    args = ap.parse_args()
    import torch

    from paper_1909_10616_b200 import tiletune as tt
    dev = torch.device("cuda:0")
    M, N, K, fam = args.M, args.N, args.K, args.fam
    tn = args.layout == "tn"
    dt = torch.bfloat16 if fam == 3 else torch.float32
    A = torch.empty((K, M) if tn else (M, K), device=dev, dtype=dt)
    B = torch.empty(K, N, device=dev, dtype=dt)
    C = torch.empty(M, N, device=dev)
    tt.fill_uniform(A, 1)
    tt.fill_uniform(B, 2)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    cfg = tuple(tuple(v) for v in json.loads(args.cfg))
    for i in range(args.n):
        flush.fill_(i & 0xFF)
        tt.gemm(A, B, C, fam, cfg, layout=tt.LAYOUT_TN if tn else tt.LAYOUT_NN)
    torch.cuda.synchronize()
    print("ok", cfg, tt.binding(tt.make_space(M, N, K, family=fam), cfg).split_tiles)


if __name__ == "__main__":
    main()

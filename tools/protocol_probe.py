"""What does the bench's cold-L2 protocol cost by itself?  (profiling aid, not a test)

Times, with CUDA events on one stream and a 256 MiB memset (the L2 flush) before each sample:
  empty      : flush | ev | ev
  torch_tiny : flush | ev | 1-element torch add | ev
  simt_tiny  : flush | ev | K1 64^3 | ev
  umma_tiny  : flush | ev | K3 256^3 (one 128x128 tile column) | ev
  umma_1024  : flush | ev | K3 1024^3 best config | ev
  umma_1024_synced : flush, host sync, then ev | K3 1024^3 | ev
  umma_1024_primed : flush | K3 256^3 (untimed: same kernel, same smem carve-out) | ev | K3 1024^3 | ev
and the same set without the flush.  Prints one JSON line per case (median of --reps, us).
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_1909_10616_b200 import tiletune as tt
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    dev = torch.device("cuda:0")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    one = torch.zeros(1, device=dev)

    def mats(M, N, K, dt):
        A = torch.empty(M, K, device=dev, dtype=dt)
        B = torch.empty(K, N, device=dev, dtype=dt)
        tt.fill_uniform(A, 1)
        tt.fill_uniform(B, 2)
        return A, B, torch.empty(M, N, device=dev)

    s64 = mats(64, 64, 64, torch.float32)
    s256 = mats(256, 256, 256, torch.bfloat16)
    s1024 = mats(1024, 1024, 1024, torch.bfloat16)
    c64 = ((2, 2, 4, 4), (8, 8), (2, 2, 4, 4))
    c256 = ((2, 1, 1, 128), (4, 64), (2, 1, 1, 128))
    c1024 = ((8, 1, 1, 128), (8, 128), (16, 1, 1, 64))
    cases = {
        "empty": lambda: None,
        "torch_tiny": lambda: one.add_(1.0),
        "simt_tiny": lambda: tt.gemm(*s64, 1, c64),
        "umma_tiny": lambda: tt.gemm(*s256, 3, c256),
        "umma_1024": lambda: tt.gemm(*s1024, 3, c1024),
    }
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    for f in cases.values():
        f()
    torch.cuda.synchronize()

    def timed(fn, do_flush, sync=False, prime=None):
        xs = []
        for r in range(reps):
            if do_flush:
                flush.fill_(r & 0xFF)
            if prime is not None:
                prime()
            if sync:
                torch.cuda.synchronize()
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            xs.append(e0.elapsed_time(e1) * 1e3)
        xs.sort()
        return xs[len(xs) // 2], xs[0]

    for flushed in (True, False):
        for name, fn in cases.items():
            med, mn = timed(fn, flushed)
            print(json.dumps({"case": name, "flush": flushed, "median_us": med, "min_us": mn}), flush=True)
        med, mn = timed(cases["umma_1024"], flushed, sync=True)
        print(json.dumps({"case": "umma_1024_synced", "flush": flushed, "median_us": med, "min_us": mn}), flush=True)
        med, mn = timed(cases["umma_1024"], flushed, prime=cases["umma_tiny"])
        print(json.dumps({"case": "umma_1024_primed", "flush": flushed, "median_us": med, "min_us": mn}), flush=True)


if __name__ == "__main__":
    main()

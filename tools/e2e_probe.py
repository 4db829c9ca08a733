"""tt_gemm_host timing (profiling aid): median / min wall time of N calls on pinned host buffers
for one config, plus pitched (2-D) copy bandwidth of the panel shapes the pipeline uses."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--cfg", default="[[16,2,1,128],[32,128],[16,1,1,256]]")
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    import torch

    from paper_1909_10616_b200 import tiletune as tt
    n = a.n
    cfg = tuple(tuple(v) for v in json.loads(a.cfg))
    Ah = torch.empty(n, n, dtype=torch.bfloat16).pin_memory()
    Bh = torch.empty(n, n, dtype=torch.bfloat16).pin_memory()
    Ch = torch.empty(n, n).pin_memory()
    Ah.copy_(torch.rand(n, n) * 2 - 1)
    Bh.copy_(torch.rand(n, n) * 2 - 1)
    ctx = tt.Context(0)
    ctx.gemm_host(Ah, Bh, Ch, tt.FAM_BF16_UMMA, cfg)
    ts = []
    for _ in range(a.reps):
        t0 = time.perf_counter()
        ctx.gemm_host(Ah, Bh, Ch, tt.FAM_BF16_UMMA, cfg)
        ts.append(time.perf_counter() - t0)
    ts.sort()
    fl = 2.0 * n ** 3
    print(json.dumps({"probe": "gemm_host", "n": n, "median_ms": ts[len(ts) // 2] * 1e3, "min_ms": ts[0] * 1e3,
                      "median_tflops": fl / ts[len(ts) // 2] / 1e12, "best_tflops": fl / ts[0] / 1e12}))
    # pitched copies: 4 column panels of B (rows of n/4 bf16) H2D, 16 C blocks D2H
    dev = torch.device("cuda:0")
    dB = torch.empty(n, n, dtype=torch.bfloat16, device=dev)
    dC = torch.empty(n, n, device=dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    from cuda.bindings import runtime as rt
    stream = torch.cuda.current_stream().cuda_stream
    H2D, D2H = rt.cudaMemcpyKind.cudaMemcpyHostToDevice, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost

    def memcpy2d_panels(q):       # cudaMemcpy2DAsync: q column panels of B (rows of n/q bf16), packed
        w = n // q * 2
        for j in range(q):
            rt.cudaMemcpy2DAsync(dB.data_ptr() + j * n * w, w, Bh.data_ptr() + j * w, n * 2, w, n, H2D, stream)

    def memcpy2d_blocks(q):       # q x q C blocks unpacked into the host matrix
        w = n // q * 4
        for i in range(q):
            for j in range(q):
                rt.cudaMemcpy2DAsync(Ch.data_ptr() + (i * (n // q) * n) * 4 + j * w, n * 4,
                                     dC.data_ptr() + (i * q + j) * (n // q) * w, w, w, n // q, D2H, stream)
    for name, fn in (("cudaMemcpy2D_h2d_4panels", lambda: memcpy2d_panels(4)),
                     ("cudaMemcpy2D_h2d_2panels", lambda: memcpy2d_panels(2)),
                     ("cudaMemcpy2D_d2h_4x4blocks", lambda: memcpy2d_blocks(4)),
                     ("cudaMemcpy2D_d2h_2x2blocks", lambda: memcpy2d_blocks(2)),
                     ("h2d_panels_2d", lambda: [dB[:, j * n // 4:(j + 1) * n // 4].copy_(Bh[:, j * n // 4:(j + 1) * n // 4], non_blocking=True) for j in range(4)]),
                     ("h2d_1d", lambda: dB.copy_(Bh, non_blocking=True)),
                     ("d2h_blocks_2d", lambda: [Ch[i * n // 4:(i + 1) * n // 4, j * n // 4:(j + 1) * n // 4].copy_(dC[i * n // 4:(i + 1) * n // 4, j * n // 4:(j + 1) * n // 4], non_blocking=True) for i in range(4) for j in range(4)]),
                     ("d2h_1d", lambda: Ch.copy_(dC, non_blocking=True))):
        best = 1e9
        for _ in range(5):
            torch.cuda.synchronize()
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e-3)
        nbytes = dB.numel() * 2 if name.startswith("h2d") else dC.numel() * 4
        print(json.dumps({"probe": name, "bytes": nbytes, "s": best, "GBps": nbytes / best / 1e9}))


if __name__ == "__main__":
    main()

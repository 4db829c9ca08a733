"""Library context for the kernel families: torch.matmul (cuBLAS / cuBLASLt) on the same shapes,
dtypes and timing protocol as bench.py (L2 flushed before every launch, CUDA events, median).
fp32 runs with TF32 disabled (CUDA-core SGEMM), tf32 with it enabled, bf16 with fp32 output
requested through out_dtype where supported (else bf16 output)."""
import json
import statistics
import sys

import torch


def timed(fn, steps=30, warmup=5):
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for _ in range(warmup):
        flush.fill_(1)
        fn()
    torch.cuda.synchronize()
    for i in range(steps):
        flush.fill_(i & 0xFF)
        ev[i][0].record()
        fn()
        ev[i][1].record()
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in ev) * 1e-3


def main():
    out = []
    for name, n, dt, tf32 in [("f32", 1024, torch.float32, False), ("f32", 2048, torch.float32, False),
                              ("f32", 4096, torch.float32, False),
                              ("tf32", 2048, torch.float32, True), ("tf32", 4096, torch.float32, True),
                              ("bf16", 1024, torch.bfloat16, False), ("bf16", 2048, torch.bfloat16, False),
                              ("bf16", 4096, torch.bfloat16, False), ("bf16", 8192, torch.bfloat16, False)]:
        torch.backends.cuda.matmul.allow_tf32 = tf32
        A = torch.rand(n, n, device="cuda", dtype=dt) * 2 - 1
        B = torch.rand(n, n, device="cuda", dtype=dt) * 2 - 1
        if dt == torch.bfloat16:
            C = torch.empty(n, n, device="cuda", dtype=torch.float32)
            try:
                torch.mm(A, B, out_dtype=torch.float32, out=C)
                fn, cdt = (lambda: torch.mm(A, B, out_dtype=torch.float32, out=C)), "fp32"
            except Exception:   # noqa: BLE001 - older torch: bf16 output
                Cb = torch.empty(n, n, device="cuda", dtype=dt)
                fn, cdt = (lambda: torch.mm(A, B, out=Cb)), "bf16"
        else:
            C = torch.empty(n, n, device="cuda", dtype=dt)
            fn, cdt = (lambda: torch.mm(A, B, out=C)), "fp32"
        t = timed(fn)
        out.append({"family": name, "n": n, "us": t * 1e6, "tflops": 2.0 * n ** 3 / t / 1e12, "c_dtype": cdt})
        print(json.dumps(out[-1]), flush=True)
    json.dump(out, open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/cublas_ref.json", "w"), indent=1)


if __name__ == "__main__":
    main()

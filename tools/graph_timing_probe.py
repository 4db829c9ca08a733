"""Does the ~5-6 us launch floor of the bench protocol come from the stream launch path?  Times the
bf16 1024^3 / 4096^3 bench configs (L2 flushed before each launch, CUDA events around the GEMM
only) with (a) stream launches (bench.py), (b) the same [flush, event, GEMM, event] sequence
captured once into a CUDA graph and replayed.  Profiling aid."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1909_10616_b200 import tiletune as tt  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for n, cfg in ((1024, ((8, 1, 1, 128), (8, 128), (16, 1, 1, 64))),
                   (4096, ((16, 2, 1, 128), (32, 128), (16, 1, 1, 256)))):
        A = torch.empty(n, n, device=dev, dtype=torch.bfloat16)
        B = torch.empty(n, n, device=dev, dtype=torch.bfloat16)
        C = torch.empty(n, n, device=dev)
        tt.fill_uniform(A, 1)
        tt.fill_uniform(B, 2)
        plan = tt.GemmPlan(A, B, C, tt.FAM_BF16_UMMA, cfg)
        s = torch.cuda.Stream()
        steps = 20
        ev = [(torch.cuda.Event(enable_timing=True, external=True), torch.cuda.Event(enable_timing=True, external=True)) for _ in range(steps)]
        out = {"n": n}
        # (a) stream launches
        with torch.cuda.stream(s):
            for _ in range(3):
                flush.fill_(1)
                plan.launch(s.cuda_stream)
            torch.cuda.synchronize()
            for i in range(steps):
                flush.fill_(i & 255)
                ev[i][0].record(s)
                plan.launch(s.cuda_stream)
                ev[i][1].record(s)
        torch.cuda.synchronize()
        t = sorted(a.elapsed_time(b) * 1e3 for a, b in ev)
        out["stream_median_us"] = t[len(t) // 2]
        # (b) graph replay of the same sequence
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(s):
                with torch.cuda.graph(g, stream=s):
                    for i in range(steps):
                        flush.fill_(i & 255)
                        ev[i][0].record(s)
                        plan.launch(s.cuda_stream)
                        ev[i][1].record(s)
            for _ in range(2):
                g.replay()
            torch.cuda.synchronize()
            g.replay()
            torch.cuda.synchronize()
            t = sorted(a.elapsed_time(b) * 1e3 for a, b in ev)
            out["graph_median_us"] = t[len(t) // 2]
        except Exception as e:  # noqa: BLE001
            out["graph_error"] = str(e)[:200]
        plan.close()
        print(json.dumps(out))


if __name__ == "__main__":
    main()

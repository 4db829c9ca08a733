"""Host<->device copy bandwidth on the box (profiling aid for tt_gemm_host / bench e2e).

H2D alone, D2H alone and both directions at once (two streams), pinned host buffers, 64 MiB
each, CUDA events; prints GB/s (1e9)."""
import json

import torch


def main():
    n = 64 << 20
    dev = torch.device("cuda:0")
    h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
    d_in = torch.empty(n, dtype=torch.uint8, device=dev)
    d_out = torch.empty(n, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(6)]

    def h2d():
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)

    for name, fns in (("h2d", [h2d]), ("d2h", [d2h]), ("both", [h2d, d2h])):
        best = 1e9
        for _ in range(8):
            torch.cuda.synchronize()
            e[0].record()
            for s in (s1, s2):
                s.wait_event(e[0])
            for f in fns:
                f()
            e[1].record(s1)
            e[2].record(s2)
            torch.cuda.current_stream().wait_event(e[1])
            torch.cuda.current_stream().wait_event(e[2])
            e[3].record()
            torch.cuda.synchronize()
            best = min(best, e[0].elapsed_time(e[3]) * 1e-3)
        print(json.dumps({"copy": name, "bytes_each": n, "s": best, "GBps_each": n / best / 1e9}))


if __name__ == "__main__":
    main()

"""Event-timed floor of a near-empty launch under bench.py's protocol (profiling aid, not a test).

    python tools/launch_floor.py

Cold = a 256 MiB memset before the launch, CUDA events around the launch only (bench.py's
protocol); warm = the same launch repeated with no flush.  Prints the median of 50 each for a
1-element torch fill (no clusters) -- the part of any small GEMM's score that is launch + event
overhead rather than the kernel's work."""
import json

import torch


def main():
    dev = torch.device("cuda:0")
    x = torch.empty(1, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for name, do_flush in (("cold", True), ("warm", False)):
        ts = []
        for r in range(50):
            if do_flush:
                flush.fill_(r & 0xFF)
            e0.record()
            x.fill_(1.0)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        ts.sort()
        print(json.dumps({"probe": "fill_1elem", "mode": name, "median_us": ts[25], "min_us": ts[0]}))
    ts = []
    for r in range(50):
        e0.record()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    print(json.dumps({"probe": "empty_event_pair", "median_us": ts[25], "min_us": ts[0]}))


if __name__ == "__main__":
    main()

"""cProfile of bench.py's tuning pass on the device (host-overhead hunt; profiling aid, not a test).

    python tools/profile_tune.py [workload] [budget]
"""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import argparse
    import torch  # noqa: F401

    import bench
    from paper_1909_10616_b200 import tiletune as tt
    wl = sys.argv[1] if len(sys.argv) > 1 else "bf16_4096"
    Mr, N, K, fam, budget = bench.WORKLOADS[wl]
    if len(sys.argv) > 2:
        budget = int(sys.argv[2])
    args = argparse.Namespace(seed=0, width=16, tune_l2_flush=True, assign="lpt", dump_tuning=None, two_phase=True)
    ctx = tt.Context(0, input_seed=1)
    sp = tt.make_space(Mr, N, K, family=fam)
    bench.tune(ctx, sp, Mr, N, K, fam, tt.LAYOUT_NN, 8, args, 1, None, 0, wl)        # warm the module
    pr = cProfile.Profile()
    t0 = time.perf_counter()
    pr.enable()
    best, rec = bench.tune(ctx, sp, Mr, N, K, fam, tt.LAYOUT_NN, budget, args, 1, None, 0, wl)
    pr.disable()
    print("wall", time.perf_counter() - t0, "tuning_wall", rec["tuning_wall_s"], "proj8",
          rec["projected_sharded_search"]["by_gpus"]["8"], "host", rec["projected_sharded_search"]["host_s"],
          "plan", rec["projected_sharded_search"]["plan_s_1gpu"])
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)


if __name__ == "__main__":
    main()

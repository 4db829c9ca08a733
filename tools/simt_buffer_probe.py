"""Same K1 config timed on the evaluator's operands (tt_measure, L2 flushed) and on freshly
allocated torch operands (bench.py's timed loop), to separate measurement noise from operand-
address effects.  python tools/simt_buffer_probe.py M 'cfg' ..."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_1909_10616_b200 import tiletune as tt
    M = int(sys.argv[1])
    ctx = tt.Context(0)
    sp = tt.make_space(M, M, M, family=1)
    dev = torch.device("cuda:0")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for c in sys.argv[2:]:
        cfg = tuple(tuple(v) for v in json.loads(c))
        ms = [ctx.measure(sp, cfg, tt.measure_opts(l2_flush=1)).cost_s * 1e6 for _ in range(3)]
        row = {"cfg": cfg, "ctx_us": [round(x, 1) for x in ms]}
        for trial in range(2):
            A = torch.empty(M, M, device=dev)
            B = torch.empty(M, M, device=dev)
            C = torch.empty(M, M, device=dev)
            tt.fill_uniform(A, seed=1)
            tt.fill_uniform(B, seed=2)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            per = []
            for i in range(13):
                flush.zero_()
                ev[0].record()
                tt.gemm(A, B, C, tt.FAM_F32_SIMT, cfg)
                ev[1].record()
                torch.cuda.synchronize()
                if i >= 3:
                    per.append(ev[0].elapsed_time(ev[1]) * 1e3)
            row[f"torch_us_{trial}"] = round(statistics.median(per), 1)
            row[f"ptrs_{trial}"] = [hex(A.data_ptr() % (1 << 24)), hex(B.data_ptr() % (1 << 24))]
            del A, B, C
        print(json.dumps(row), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()

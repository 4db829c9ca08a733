"""bench.py contract pieces that run without a GPU: the reference arm's JSON line and argument
validation (the GPU arm is exercised on the B200 by the driver and tools/gpu_round.sh)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                        "--warmup", "3", "--ref-rows", "4", "--workload", "f32_512"],
                       capture_output=True, text=True, timeout=600, check=True)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e", "impl"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_reference_arm_nonzero_rank_is_silent():
    env = dict(os.environ, RANK="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "3"], capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0 and r.stdout.strip() == ""


def test_warmup_floor():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--warmup", "1"], capture_output=True,
                       text=True, timeout=120)
    assert r.returncode != 0


def test_sharded_projection_of_a_recorded_search():
    # bench.project_sharded on a one-rank search with fake two-phase measurements (no GPU): the
    # projection replays the evaluator's plans for G = 2, 4, 8 and reports every variant
    import hashlib
    import time

    import bench
    from paper_1909_10616_b200 import dist as tdist
    from paper_1909_10616_b200 import tiletune as tt

    M = 4096
    sp = tt.make_space(M, M, M, family=tt.FAM_BF16_UMMA)

    def cost(s):
        h = hashlib.sha256(repr(s).encode()).digest()
        return 9e-5 + int.from_bytes(h[:4], "little") / 2 ** 32 * 3e-4

    def measure_set(states, mine):
        return [cost(s) if m else 0.0 for s, m in zip(states, mine)], \
               [11 * (cost(s) + 7e-5) if m else 0.0 for s, m in zip(states, mine)]

    def measure_phase(states, mine, phase, probes):
        vals = [cost(s) if m else 0.0 for s, m in zip(states, mine)]
        secs = [(cost(s) + 7e-5) * (1 if phase == 1 else 10) if m else 0.0 for s, m in zip(states, mine)]
        return vals, [phase == 2] * len(states), secs

    ev = tdist.ShardedEvaluator(measure_set=measure_set, measure_phase=measure_phase, space=sp)
    t0 = time.perf_counter()
    res = tt.gbfs_search(M, M, M, 128, tt.search_opts(family=tt.FAM_BF16_UMMA, seed=0, width=16), batch=ev)
    wall = time.perf_counter() - t0 + sum(map(sum, ev.round_times))
    assert res.evals == 128 and "two-phase" in ev.round_modes
    assert all(len(p[0]) == len(st) for p, st, md in zip(ev.round_phase1, ev.round_states, ev.round_modes)
               if md == "two-phase")
    pr = bench.project_sharded(ev, wall, sp, lambda b: 1e-3, 30e-6)
    assert pr["round_sizes"] == [len(r) for r in ev.round_states] and pr["rounds"] == ev.rounds
    for G in ("2", "4", "8"):
        e = pr["by_gpus"][G]
        for v in ("two_phase", "lpt", "dynamic", "static"):
            assert 1.0 < e[v + "_speedup"] <= int(G) + 1e-9
        assert e["two_phase_rounds"] >= 1
    assert pr["by_gpus"]["8"]["two_phase_speedup"] > pr["by_gpus"]["2"]["two_phase_speedup"]

"""CLI harness on the synthetic backend: paper counts, CSV schema, summary
statistics recomputed from the trace, determinism apart from wall clock."""
import csv
import json
import subprocess
import sys

import pytest

from paper_1909_10616_b200 import cli


def run(*args):
    return subprocess.run([sys.executable, "-m", "paper_1909_10616_b200.cli", *args], capture_output=True,
                          text=True, check=True).stdout


@pytest.mark.parametrize("dim,count", [(512, "484000"), (1024, "899756"), (2048, "1589952")])
def test_count_paper_values(dim, count):
    # S:461-462 / P:375
    assert run("count", "--m", str(dim), "--k", str(dim), "--n", str(dim)).strip() == count


def test_compare_csv_summary_determinism(tmp_path):
    out1, out2 = str(tmp_path / "a"), str(tmp_path / "b")
    args = ["compare", "--m", "64", "--k", "64", "--n", "64", "--backend", "synthetic", "--seeds", "0-3",
            "--max-evals", "150"]
    run(*args, "--out", out1)
    run(*args, "--out", out2)
    rows1 = list(csv.DictReader(open(out1 + ".csv")))
    rows2 = list(csv.DictReader(open(out2 + ".csv")))
    strip = lambda rows: [{k: v for k, v in r.items() if k != "wall_clock_s"} for r in rows]
    assert strip(rows1) == strip(rows2)
    summ = json.load(open(out1 + ".json"))
    for strat in ("gbfs", "na2c", "random"):
        per_seed = {}
        for r in rows1:
            if r["strategy"] != strat:
                continue
            per_seed.setdefault(r["trial_seed"], []).append(r)
        bests = []
        for seed, rs in per_seed.items():
            b = [float(r["best_so_far_s"]) for r in rs]
            assert all(x >= y for x, y in zip(b, b[1:]))
            f = [float(r["fraction_explored"]) for r in rs]
            assert all(x < y for x, y in zip(f, f[1:]))
            assert cli.decode(rs[-1]["config"])                   # config text parses back
            bests.append(b[-1])
        assert summ["strategies"][strat]["best_cost"] == cli.box(bests)


def test_decode_errors():
    with pytest.raises(ValueError):
        cli.decode('{"m":[32,1.5,1,1],"k":[256,4],"n":[32,32,1,1]}')
    with pytest.raises(ValueError):
        cli.decode('{"m":[32,32,1],"k":[256,4],"n":[32,32,1,1]}')
    assert cli.decode('{"m":[32,32,1,1],"k":[256,4],"n":[32,32,1,1]}') == ((32, 32, 1, 1), (256, 4), (32, 32, 1, 1))


def test_compare_refuses_single_strategy(tmp_path):
    r = subprocess.run([sys.executable, "-m", "paper_1909_10616_b200.cli", "compare", "--m", "64", "--k", "64", "--n",
                        "64", "--backend", "synthetic", "--strategies", "gbfs", "--out", str(tmp_path / "x")],
                       capture_output=True, text=True)
    assert r.returncode != 0


def test_resume_from_trace_is_exact(tmp_path):
    # the trace is the checkpoint.  A 120-eval run resumed to 250 == a direct 250 run.
    base = ["tune", "--m", "64", "--k", "64", "--n", "64", "--backend", "synthetic", "--seeds", "3"]
    for strat in ("gbfs", "na2c", "random"):
        a, b, c = (str(tmp_path / f"{strat}_{x}") for x in "abc")
        run(*base, "--strategy", strat, "--max-evals", "120", "--out", a)
        run(*base, "--strategy", strat, "--max-evals", "250", "--resume", a + ".csv", "--out", b)
        run(*base, "--strategy", strat, "--max-evals", "250", "--out", c)
        key = lambda p: [(r["eval_index"], r["config"], r["cost_s"]) for r in csv.DictReader(open(p + ".csv"))]
        assert key(b) == key(c) and len(key(b)) == 250

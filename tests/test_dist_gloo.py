"""Multi-process (gloo, world size 2, CPU) coverage of the sharded search:
every rank runs the identical G-BFS / N-A2C, candidates are measured round-robin over ranks and the
costs are all-gathered; the traversal must equal the single-process oracle traversal."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from oracle import costs, gbfs as ogbfs, na2c as ona2c, space
from oracle.space import Spec
from paper_1909_10616_b200 import dist as tdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, algo, out, dynamic=False):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1909_10616_b200 import dist as tdist
    from paper_1909_10616_b200 import tiletune as tt

    sp = Spec(64, 64, 64)
    measured = []

    def measure_one(s):
        measured.append(s)
        return costs.t2_cost(sp, s)

    ev = tdist.ShardedEvaluator(measure_one, store=tdist.default_store() if dynamic else None)
    assert (ev.store is not None) == dynamic
    if algo == "gbfs":
        res = tt.gbfs_search(64, 64, 64, 300, tt.search_opts(seed=4, width=8), batch=ev)
    else:
        res = tt.na2c_search(64, 64, 64, 200, tt.search_opts(seed=4, epsilon=0.0), batch=ev)
    row_ranges = tdist.row_shard(8192, world, rank)
    out[rank] = ([(r["state"], r["cost"]) for r in res.trace], len(measured), ev.rounds, row_ranges)
    dist.destroy_process_group()


@pytest.mark.parametrize("algo,dynamic", [("gbfs", False), ("na2c", False), ("gbfs", True), ("na2c", True)])
def test_sharded_search_matches_oracle(algo, dynamic):
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), algo, out, dynamic), nprocs=world, join=True)
    sp = Spec(64, 64, 64)
    tab = costs.table(sp, lambda s: costs.t2_cost(sp, s))
    if algo == "gbfs":
        o = ogbfs.gbfs(sp, ogbfs.table_source(sp, tab), budget=300, rho=5, seed=4, width=8)
    else:
        o = ona2c.na2c(sp, ogbfs.table_source(sp, tab), budget=200, params=ona2c.Params(epsilon=0.0), seed=4)
    ref = [(r.state, r.cost) for r in o.trace]
    t0, n0, rounds0, rr0 = out[0]
    t1, n1, rounds1, rr1 = out[1]
    assert t0 == t1 == ref                                 # identical traversal on every rank = oracle
    assert n0 + n1 == len(ref)                             # each candidate measured exactly once
    if not dynamic:
        assert abs(n0 - n1) <= rounds0                     # round-robin balance
    assert rr0 == (0, 4096) and rr1 == (4096, 8192)        # exact row partition

def test_projection():
    rt = [[1.0], [1.0, 2.0, 3.0, 4.0], [0.5] * 8]
    assert tdist.projected_sharded_wall(rt, 1) == 1.0 + 10.0 + 4.0
    # G = 2: round 2 shares (1+3, 2+4) -> 6; round 3 -> 2.0
    assert tdist.projected_sharded_wall(rt, 2) == 1.0 + 6.0 + 2.0
    assert tdist.projected_sharded_wall(rt, 8, per_round_s=0.1) == 1.1 + 4.1 + 0.6
    # dynamic: list scheduling in index order, each candidate to the first free rank
    assert tdist.projected_sharded_wall([[4.0, 1.0, 1.0, 1.0, 1.0]], 2, dynamic=True) == 4.0
    assert tdist.projected_sharded_wall([[4.0, 1.0, 1.0, 1.0, 1.0]], 2) == 6.0

"""Scenario sharding across ranks: world_size 2 over gloo on CPU.

The multi-GPU path has no data-path collective: each rank builds its own
contiguous rows of the seeded batch and solves them; only the timing
(max over ranks) and counters (sum) cross ranks. This test runs that host
logic with two gloo processes and checks the shards reassemble the batch.
"""

import os
import socket

import numpy as np
import torch.multiprocessing as mp

import paper_2605_14103_b200 as pf
from paper_2605_14103_b200 import shard
from paper_2605_14103_b200.fixtures import load_transmission


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, total, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    r, _, w = shard.dist_env()
    net = load_transmission("case118")
    m = pf.build_transmission_model(net)
    base = pf.transmission_base(net, m.part)
    a, b = shard.shard_range(total, r, w)
    spec = pf.ScenarioSpec(count=total, seed=1010)
    p, _ = pf.make_scenario_arrays(base, spec, start=a, count=b - a)
    t = shard.max_over_ranks(1.0 + r)
    n = shard.sum_over_ranks(b - a)
    out[r] = (a, b, p, t, n)
    dist.destroy_process_group()


def test_two_rank_shards_reassemble():
    total = 11
    port = _free_port()
    with mp.Manager() as man:
        out = man.dict()
        mp.spawn(_worker, args=(2, port, total, out), nprocs=2, join=True)
        res = dict(out)
    (a0, b0, p0, t0, n0), (a1, b1, p1, t1, n1) = res[0], res[1]
    assert (a0, b0, a1, b1) == (0, 6, 6, 11)
    assert t0 == t1 == 2.0 and n0 == n1 == total
    net = load_transmission("case118")
    m = pf.build_transmission_model(net)
    full, _ = pf.make_scenario_arrays(pf.transmission_base(net, m.part),
                                      pf.ScenarioSpec(count=total, seed=1010))
    np.testing.assert_array_equal(np.concatenate([p0, p1]), full)


def test_shard_range_partitions():
    for total in (1, 7, 64, 1000):
        for world in (1, 2, 3, 8):
            rng = [shard.shard_range(total, r, world) for r in range(world)]
            assert rng[0][0] == 0 and rng[-1][1] == total
            assert all(rng[i][1] == rng[i + 1][0] for i in range(world - 1))

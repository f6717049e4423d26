"""CPU, world_size 2 over gloo: the multi-GPU plumbing of the Solver.

Each rank builds its contiguous ant shard (here with the oracle's restatement
of the device stream, keyed by GLOBAL ant id), the colony is all-gathered
with distributed.gather_colony, and every rank then derives the identical
elite order and deposit — the replicated-pheromone scheme of DESIGN.md §6.
The result must equal a single-process run over all ants (R-invariance).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import fastpath, reference_port as ref


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _colony(n: int):
    coords = np.random.default_rng(42).uniform(0, 1000, (n, 2))
    dist_m, eta = ref.instance_arrays(coords)
    p = ref.transition(ref.initial_tau(n, 1.0), eta, 1.0, 2.0)
    return dist_m, fastpath.selection_table(p, 1.0)


def _worker(rank: int, world: int, port: int, m: int, n: int, out_dir: str) -> None:
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2404_04895_b200 import distributed

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dist_m, w = _colony(n)
        sh = distributed.shard_ants(m, rank, world)
        local = np.zeros((sh.per_rank, n), dtype=np.int32)
        costs = np.zeros(sh.per_rank)
        tours = fastpath.build_tours(w, 3, 1, np.arange(sh.offset, sh.offset + sh.count))
        local[:sh.count] = tours
        costs[:sh.count] = ref.lengths(tours, dist_m)
        tours_all = torch.zeros((m, n), dtype=torch.int32)
        costs_all = torch.zeros(m, dtype=torch.float64)
        pad_t = torch.zeros((world * sh.per_rank, n), dtype=torch.int32) if m % world else None
        pad_c = torch.zeros(world * sh.per_rank, dtype=torch.float64) if m % world else None
        distributed.gather_colony(torch.from_numpy(local), torch.from_numpy(costs), sh, tours_all, costs_all,
                                  None, pad_t, pad_c)
        order = ref.elite_ranks(costs_all.numpy(), max(1, m // 10))
        delta = ref.deposit(tours_all.numpy()[order].astype(np.int64), costs_all.numpy()[order], n)
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), tours=tours_all.numpy(), costs=costs_all.numpy(),
                 order=order, delta=delta)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("m", [12, 7])  # even and uneven shards
def test_sharded_colony_equals_single_process(tmp_path, m):
    n, world = 23, 2
    mp.start_processes(_worker, args=(world, _free_port(), m, n, str(tmp_path)), nprocs=world,
                       start_method="spawn", join=True)
    dist_m, w = _colony(n)
    want = fastpath.build_tours(w, 3, 1, np.arange(m))
    want_costs = ref.lengths(want, dist_m)
    ranks = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    for r in ranks:
        assert np.array_equal(r["tours"], want)
        assert np.array_equal(r["costs"], want_costs)
    # every rank applies the identical elite deposit: replicated pheromone
    assert np.array_equal(ranks[0]["order"], ranks[1]["order"])
    assert np.array_equal(ranks[0]["delta"], ranks[1]["delta"])

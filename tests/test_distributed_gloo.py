"""CPU, world_size 2-4 over gloo: the multi-GPU plumbing of the Solver.

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
        # costs-first exchange (the Solver's path): lengths, identical ranking,
        # then only the k elite tours, each rank filling the rows it owns
        k = max(1, m // 10)
        costs2 = torch.zeros(m, dtype=torch.float64)
        distributed.gather_costs(torch.from_numpy(costs), sh, costs2, None,
                                 torch.zeros(world * sh.per_rank, dtype=torch.float64) if m % world else None)
        order2 = ref.elite_ranks(costs2.numpy(), k)
        elite = np.zeros((k, n), dtype=np.int32)
        for r, a in enumerate(order2):  # what taco_shard_elites does on the device
            if sh.offset <= a < sh.offset + sh.count:
                elite[r] = local[a - sh.offset]
        elite_t = distributed.share_elites(torch.from_numpy(elite))
        delta2 = ref.deposit(elite_t.numpy().astype(np.int64), costs2.numpy()[order2], n)
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), tours=tours_all.numpy(), costs=costs_all.numpy(),
                 order=order, delta=delta, costs2=costs2.numpy(), order2=order2, elite=elite_t.numpy(),
                 delta2=delta2)
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
    # the costs-first exchange reaches the same elites and deposit with k x n traffic
    order = ref.elite_ranks(want_costs, max(1, m // 10))
    for r in ranks:
        assert np.array_equal(r["costs2"], want_costs)
        assert np.array_equal(r["order2"], order)
        assert np.array_equal(r["elite"], want[order])
        assert np.array_equal(r["delta2"], ranks[0]["delta"])


def _row_worker(rank: int, world: int, port: int, n: int, out_dir: str) -> None:
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2404_04895_b200 import distributed

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # each rank runs the row update on its rows only (here: the oracle's
        # row normalization), the table rows are then gathered in place
        tau = ref.initial_tau(n, 1.0) + np.random.default_rng(3).uniform(0, 1, (n, n))
        _, eta = ref.instance_arrays(np.random.default_rng(42).uniform(0, 1000, (n, 2)))
        part = distributed.row_partition(n, rank, world)
        p_full = ref.transition(tau, eta, 1.0, 2.0)
        buf = torch.full((part.rows, n), -1.0, dtype=torch.float64)
        buf[part.begin:part.end] = torch.from_numpy(p_full[part.begin:part.end])
        distributed.gather_rows(buf, part)
        # status: rank 1 saw (NO_CANDIDATE, ant 5), rank 0 (NO_CANDIDATE, ant 9)
        # and, in a second round, rank 0 an UNDERFLOW at row 40 — highest code,
        # then smallest row, on every rank
        st = torch.tensor([2, 9 if rank == 0 else 5, 0, rank], dtype=torch.int32)
        distributed.share_status(st)
        st2 = torch.tensor([1, 40, 0, 0] if rank == 0 else [0, 2**31 - 1, 0, 0], dtype=torch.int32)
        distributed.share_status(st2)
        st3 = torch.tensor([0, 2**31 - 1, 0, 0], dtype=torch.int32)
        distributed.share_status(st3)
        np.savez(os.path.join(out_dir, f"rows{rank}.npz"), p=buf.numpy()[:n], want=p_full, st=st.numpy(),
                 st2=st2.numpy(), st3=st3.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 23), (3, 10), (4, 3)])  # uneven chunks, an empty rank
def test_row_partitioned_update_gathers_every_row(tmp_path, world, n):
    from paper_2404_04895_b200.distributed import row_partition

    parts = [row_partition(n, r, world) for r in range(world)]
    assert parts[0].begin == 0 and parts[-1].end == n
    assert all(a.end == b.begin for a, b in zip(parts, parts[1:]))
    assert all(p.end - p.begin <= p.chunk for p in parts)
    mp.start_processes(_row_worker, args=(world, _free_port(), n, str(tmp_path)), nprocs=world,
                       start_method="spawn", join=True)
    for r in range(world):
        got = np.load(tmp_path / f"rows{r}.npz")
        assert np.array_equal(got["p"], got["want"])
        assert got["st"][:2].tolist() == [2, 5] and got["st"][3] == r  # the local stop flag stays
        assert got["st2"][:2].tolist() == [1, 40]
        assert got["st3"][:2].tolist() == [0, 2**31 - 1]

"""GPU: the sharded Solver with real kernels, two ranks in two processes.

Only one GPU is available to the test, so both ranks use cuda:0 and exchange
tours over gloo (host-side collective: no kernel ever waits on another
rank's kernel).  The sharded run must equal the single-process run bit for bit
(R-invariance: the device stream is keyed by global ant id; the deposit is
identical on every rank), with the pheromone update replicated (every rank
updates all rows) or row-partitioned (each rank updates its rows and the
construction tables are all-gathered) — for the sorted table, the dense table
and RW's P.  A failure seen by one rank's ants is raised by every rank.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

N, M, ITERS = 71, 37, 4  # m and n not divisible by the world size: padded gathers

# (update, construct, selection)
CASES = [("replicated", "sorted", "adair"), ("partitioned", "sorted", "adair"),
         ("partitioned", "dense", "ir"), ("partitioned", "sorted", "rw")]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _params(selection="adair"):
    import paper_2404_04895_b200 as taco

    return taco.AcoParams(m=M, k=5, selection=selection, seed=17,
                          gamma_schedule=taco.GammaSchedule(1.5, 1.0, ITERS))


def _run(s):
    tours, taus = [], []
    for _ in range(ITERS):
        s.step()
        tours.append(s.last_batch().tours)
        taus.append(s.pheromone().tau)
    return np.stack(tours), np.stack(taus), s.best()


def _inst():
    import paper_2404_04895_b200 as taco

    return taco.euclidean_instance(np.random.default_rng(5).uniform(0, 1000, (N, 2)))


def _worker(rank: int, world: int, port: int, out_dir: str) -> None:
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_2404_04895_b200 as taco

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for i, (update, construct, selection) in enumerate(CASES):
            s = taco.Solver(_inst(), _params(selection), construct=construct, update=update)
            assert s.shard.world == world and s.shard.rank == rank
            assert s.partitioned == (update == "partitioned")
            tours, taus, best = _run(s)
            ckpt = s.checkpoint()["tau"]
            np.savez(os.path.join(out_dir, f"case{i}_rank{rank}.npz"), tours=tours, tau=taus,
                     best_tour=best[0], best_len=best[1], ckpt=ckpt)
        # a failure recorded by rank 1 alone (its ant 5 found no candidate)
        # reaches rank 0's status at the next update: both ranks raise it
        s = taco.Solver(_inst(), _params(), update="partitioned")
        s.step()
        if rank == 1:
            s.status[0:2].copy_(torch.tensor([taco._lib.TACO_NO_CANDIDATE, 5], dtype=torch.int32))
        raised = 0
        try:
            s.step()
        except AssertionError:
            raised = int(s.status[1].item() == 5)
        np.save(os.path.join(out_dir, f"raised_rank{rank}.npy"), np.array(raised))
    finally:
        dist.destroy_process_group()


def test_two_rank_solver_equals_single_gpu(tmp_path):
    import paper_2404_04895_b200 as taco

    mp.start_processes(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, start_method="spawn", join=True)
    for i, (update, construct, selection) in enumerate(CASES):
        tours, taus, best = _run(taco.Solver(_inst(), _params(selection), construct=construct))
        for r in range(2):
            got = np.load(tmp_path / f"case{i}_rank{r}.npz")
            assert np.array_equal(got["tours"], tours), (update, construct, selection, r)
            assert np.array_equal(got["tau"], taus), (update, construct, selection, r)
            assert np.array_equal(got["ckpt"], taus[-1])
            assert float(got["best_len"]) == best[1]
    for r in range(2):
        assert int(np.load(tmp_path / f"raised_rank{r}.npy")) == 1

"""GPU: the sharded Solver with real kernels, two ranks in two processes.

Only one GPU is available to the test, so both ranks use cuda:0 and exchange
tours over gloo (host-side collective: no kernel ever waits on another
rank's kernel).  The sharded run must equal the single-process run bit for bit
(R-invariance: the device stream is keyed by global ant id; every rank applies
the identical deposit to its replicated pheromone).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

N, M, ITERS = 70, 37, 4  # m not divisible by the world size: padded gather


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _params():
    import paper_2404_04895_b200 as taco

    return taco.AcoParams(m=M, k=5, selection="adair", seed=17,
                          gamma_schedule=taco.GammaSchedule(1.5, 1.0, ITERS))


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
        s = taco.Solver(_inst(), _params())
        assert s.shard.world == world and s.shard.rank == rank
        tours, taus = [], []
        for _ in range(ITERS):
            s.step()
            tours.append(s.last_batch().tours)
            taus.append(s.pheromone().tau)
        best = s.best()
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), tours=np.stack(tours), tau=np.stack(taus),
                 best_tour=best[0], best_len=best[1])
    finally:
        dist.destroy_process_group()


def test_two_rank_solver_equals_single_gpu(tmp_path):
    import paper_2404_04895_b200 as taco

    mp.start_processes(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, start_method="spawn", join=True)
    s = taco.Solver(_inst(), _params())
    tours, taus = [], []
    for _ in range(ITERS):
        s.step()
        tours.append(s.last_batch().tours)
        taus.append(s.pheromone().tau)
    for r in range(2):
        got = np.load(tmp_path / f"rank{r}.npz")
        assert np.array_equal(got["tours"], np.stack(tours))
        assert np.array_equal(got["tau"], np.stack(taus))
        assert float(got["best_len"]) == s.best()[1]

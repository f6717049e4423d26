"""Ant sharding across the GPUs of one box (one process per GPU).

Ants are independent within an iteration (colony.py:126-152; chunking is
bit-invisible, tests/test_colony.py:120-129 of the reference), and the device
stream is keyed by the GLOBAL ant index, so a rank that builds ants
[offset, offset + count) produces exactly the rows a single GPU would.  One
exchange per iteration: the tours and lengths are all-gathered, then every
rank runs the identical elite sort, deposit and P rebuild on replicated
state — no n x n all-reduce.  The helpers work on any torch.distributed
backend (NCCL on the B200 box, gloo for the CPU tests).

The Solver uses the costs-first form: all-gather the m lengths,
rank them identically on every rank, then assemble only the k elite tours
with one SUM all-reduce of a k x n buffer in which each rank filled the rows
it owns (taco_shard_elites) — k·n·4 bytes instead of m·n·4 (10x less at
k = m/10).  ``gather_colony`` (all tours) remains for ``last_batch()``.

Row-partitioned update (optional; replicated is the default): the deposit is identical
on every rank, and the row update is independent per row (colony.py:27-60,
evaporation + row normalization), so rank r updates only rows
[r·nr, (r+1)·nr) of tau, P and the selection table (``row_partition``) and
the construction input is then all-gathered in place (``gather_rows``):
n²·4·(R-1)/R bytes in, (R-1)/R of the update work saved.  ``share_status``
keeps the fail-stop status words identical on every rank.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


@dataclass(frozen=True)
class AntShard:
    """Contiguous slice of the colony owned by one rank."""

    rank: int
    world: int
    m: int
    offset: int
    count: int
    per_rank: int  # padded slice length used by the all-gather


def shard_ants(m: int, rank: int, world: int) -> AntShard:
    """Split m ants into `world` contiguous slices; the first m % world ranks
    take one extra ant."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    if m < world:
        raise ValueError(f"need at least one ant per rank (m={m}, world={world})")
    base, extra = divmod(m, world)
    offset = rank * base + min(rank, extra)
    count = base + (1 if rank < extra else 0)
    return AntShard(rank, world, m, offset, count, base + (1 if extra else 0))


def gather_index(m: int, world: int) -> torch.Tensor | None:
    """Rows of the padded gather buffer that hold real ants, in global order
    (None when m divides evenly and the buffer is already compact)."""
    if m % world == 0:
        return None
    rows = []
    for r in range(world):
        s = shard_ants(m, r, world)
        rows.extend(range(r * s.per_rank, r * s.per_rank + s.count))
    return torch.tensor(rows, dtype=torch.long)


def _all_gather_into(out: torch.Tensor, inp: torch.Tensor, group) -> None:
    try:
        dist.all_gather_into_tensor(out, inp, group=group)
    except (RuntimeError, NotImplementedError, AttributeError):
        # backends without the fused form (older gloo): list all-gather
        parts = list(out.chunk(dist.get_world_size(group)))
        dist.all_gather(parts, inp, group=group)


def gather_colony(local_tours: torch.Tensor, local_costs: torch.Tensor, shard: AntShard,
                  tours_all: torch.Tensor, costs_all: torch.Tensor, group=None,
                  pad_tours: torch.Tensor | None = None,
                  pad_costs: torch.Tensor | None = None) -> tuple[torch.Tensor, torch.Tensor]:
    """All-gather every rank's tours (per_rank x n) and lengths into the
    global (m x n) / (m,) buffers, in global ant order.

    ``local_tours``/``local_costs`` must be per_rank rows long (rows past
    ``shard.count`` are padding).  When m % world != 0 the gather lands in
    ``pad_tours``/``pad_costs`` (world * per_rank rows) and is compacted.
    """
    if shard.m % shard.world == 0:
        _all_gather_into(tours_all, local_tours, group)
        _all_gather_into(costs_all, local_costs, group)
        return tours_all, costs_all
    if pad_tours is None or pad_costs is None:
        raise ValueError("uneven shards need padded gather buffers")
    _all_gather_into(pad_tours, local_tours, group)
    _all_gather_into(pad_costs, local_costs, group)
    idx = gather_index(shard.m, shard.world).to(pad_tours.device)
    torch.index_select(pad_tours, 0, idx, out=tours_all)
    torch.index_select(pad_costs, 0, idx, out=costs_all)
    return tours_all, costs_all


def gather_costs(local_costs: torch.Tensor, shard: AntShard, costs_all: torch.Tensor, group=None,
                 pad_costs: torch.Tensor | None = None) -> torch.Tensor:
    """All-gather every rank's tour lengths into the global (m,) buffer in
    global ant order (first half of the costs-first exchange)."""
    if shard.m % shard.world == 0:
        _all_gather_into(costs_all, local_costs, group)
        return costs_all
    if pad_costs is None:
        raise ValueError("uneven shards need a padded gather buffer")
    _all_gather_into(pad_costs, local_costs, group)
    idx = gather_index(shard.m, shard.world).to(pad_costs.device)
    torch.index_select(pad_costs, 0, idx, out=costs_all)
    return costs_all


def share_elites(elite_tours: torch.Tensor, group=None) -> torch.Tensor:
    """Second half: every rank filled the elite rows it owns (zeros elsewhere);
    an integer SUM all-reduce leaves every elite tour on every rank, exactly."""
    dist.all_reduce(elite_tours, op=dist.ReduceOp.SUM, group=group)
    return elite_tours


@dataclass(frozen=True)
class RowPartition:
    """Rows [begin, end) of an n-row table owned by one rank; every rank's
    chunk is `chunk` rows (the buffers carry world * chunk rows, the tail
    rows past n are padding) so one equal-size all-gather moves them."""

    rank: int
    world: int
    n: int
    chunk: int
    begin: int
    end: int

    @property
    def rows(self) -> int:
        return self.world * self.chunk


def row_partition(n: int, rank: int, world: int) -> RowPartition:
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    chunk = -(-n // world)
    return RowPartition(rank, world, n, chunk, min(n, rank * chunk), min(n, (rank + 1) * chunk))


def gather_rows(buf: torch.Tensor, part: RowPartition, group=None) -> torch.Tensor:
    """In-place all-gather of a row-partitioned (world * chunk, ...) buffer:
    afterwards every rank holds every rank's rows."""
    if buf.shape[0] != part.rows or not buf.is_contiguous():
        raise ValueError(f"need a contiguous buffer of {part.rows} rows, got {tuple(buf.shape)}")
    c = part.chunk
    raw = buf.view(torch.uint8)  # as bytes: gloo / NCCL have no uint16 (the sorted table's indices)
    _all_gather_into(raw, raw[part.rank * c:(part.rank + 1) * c], group)
    return buf


_INT32_MAX = 2**31 - 1


def share_status(status: torch.Tensor, group=None) -> torch.Tensor:
    """Make the 4 fail-stop status words (include/taco.h) identical on every
    rank without a host sync: one MAX all-reduce of
    (code << 32 | INT32_MAX - row) — the highest code wins, then the smallest
    row / ant.  status[3] (the local stop flag) is left alone."""
    key = status[0:1].to(torch.int64) * (1 << 32) + (_INT32_MAX - status[1:2].to(torch.int64))
    dist.all_reduce(key, op=dist.ReduceOp.MAX, group=group)
    status[0:1].copy_(key >> 32)
    status[1:2].copy_(_INT32_MAX - (key & 0xFFFFFFFF))
    return status

"""Multi-GPU partitioning of the encode: every generation is
independent, and inside a generation every byte column m is independent
(B[:, m] depends only on A[:, m] and C, Eq. 2), so ranks split
the job by generation or by packet byte range and never exchange data on the
hot path.  One process per GPU; no collective except the benchmark's
barrier / max-over-ranks timing.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    g0: int          # first generation (absolute index in the global job)
    g1: int          # one past the last generation
    m0: int          # first byte column of every packet
    m1: int          # one past the last byte column

    @property
    def generations(self) -> int:
        return self.g1 - self.g0

    @property
    def columns(self) -> int:
        return self.m1 - self.m0


def generation_range(batch: int, world: int, rank: int) -> tuple:
    """Contiguous, balanced split of `batch` generations (sizes differ by <= 1)."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return batch * rank // world, batch * (rank + 1) // world


def byte_range(M: int, world: int, rank: int, align: int = 16) -> tuple:
    """Split of the packet byte range with interior boundaries on multiples of
    `align` (so every shard keeps 16-B aligned rows when M is)."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    units = -(-M // align)
    u0, u1 = units * rank // world, units * (rank + 1) // world
    return min(M, u0 * align), min(M, u1 * align)


def plan(batch: int, M: int, world: int, rank: int, by: str = "generation",
         weak: bool = False) -> Shard:
    """Shard of rank `rank`.

    by="generation": strong scaling splits `batch` generations; weak scaling
    gives every rank `batch` generations of a world*batch job.
    by="bytes": every rank holds all generations and columns [m0, m1)."""
    if by == "generation":
        if weak:
            return Shard(rank, world, rank * batch, (rank + 1) * batch, 0, M)
        g0, g1 = generation_range(batch, world, rank)
        return Shard(rank, world, g0, g1, 0, M)
    if by == "bytes":
        m0, m1 = byte_range(M, world, rank)
        return Shard(rank, world, 0, batch, m0, m1)
    raise ValueError(by)

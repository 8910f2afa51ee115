"""Range sharding over ranks and the one cross-device step: reducing the tiny
result vector with torch.distributed (NCCL over NVLink on B200, gloo in CPU tests).

PAPER.md:354 ("--gpus=i flag that distributes work across the requested GPUs")
leaves the policy open; here the even range is cut into word-aligned strips that
ranks take round-robin (strip r, r + R, r + 2R, ...), so the slow growth of the
per-n cost with n is spread evenly.  Results over
disjoint ranges compose by SUM (counts, hist, sum_pmin, checksum halves), MIN
(first unresolved n) and MAX (max key), so no halo or data exchange is needed.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import gb

STRIP_ALIGN = 1 << 20     # integers; strips start on multiples (U-word and tile friendly)


def plan_strips(lo: int, hi: int, n_strips: int, align: int = STRIP_ALIGN) -> list[tuple[int, int]]:
    """Cut [lo, hi) into n_strips consecutive half-open strips with interior
    boundaries on multiples of `align` (empty strips are dropped)."""
    if hi <= lo:
        return []
    n_strips = max(1, n_strips)
    span = hi - lo
    cuts = [lo]
    for i in range(1, n_strips):
        c = lo + span * i // n_strips
        c = (c // align) * align
        cuts.append(min(max(c, cuts[-1]), hi))
    cuts.append(hi)
    return [(a, b) for a, b in zip(cuts[:-1], cuts[1:]) if b > a]


def rank_strips(strips: list[tuple[int, int]], rank: int, world: int) -> list[tuple[int, int]]:
    return strips[rank::world]


def reduce_result(result: torch.Tensor, group=None) -> None:
    """In-place cross-rank reduction of a FINALIZED result vector (int64)."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return
    s1 = result[gb.R_EVENS:gb.R_SUM_PMIN + 1]            # SUM fields 1..5
    s2 = result[gb.R_HIST:gb.R_HIST + gb.NBINS]          # SUM hist
    mx = torch.stack([result[gb.R_MAX_KEY], result[gb.R_MAX_PMIN_RAW]])
    mn = result[gb.R_FIRST_UNRESOLVED_N:gb.R_FIRST_UNRESOLVED_N + 1]
    sums = torch.cat([s1, s2])
    dist.all_reduce(sums, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=group)
    dist.all_reduce(mn, op=dist.ReduceOp.MIN, group=group)
    result[gb.R_EVENS:gb.R_SUM_PMIN + 1] = sums[:s1.numel()]
    result[gb.R_HIST:gb.R_HIST + gb.NBINS] = sums[s1.numel():]
    result[gb.R_MAX_KEY] = mx[0]
    result[gb.R_MAX_PMIN_RAW] = mx[1]
    result[gb.R_FIRST_UNRESOLVED_N] = mn[0]


def verify_sharded(verifier, lo: int, hi: int, rank: int, world: int, strips_per_rank: int = 32,
                   p_max: int | None = None, result: torch.Tensor | None = None,
                   reduce: bool = True, group=None) -> torch.Tensor:
    """This rank's share of [lo, hi) through libgb, then (optionally) the NCCL reduction."""
    r = verifier.new_result() if result is None else result
    for a, b in rank_strips(plan_strips(lo, hi, strips_per_rank * world), rank, world):
        verifier.verify(a, b, r, p_max=p_max)
    verifier.finalize(r)
    if reduce:
        reduce_result(r, group)
    return r

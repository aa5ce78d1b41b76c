"""Data parallelism over views.

Training views are independent units of the step: each rank renders its own views, and
the only exchange is ONE all-reduce (sum) of the compact active-gradient rows
grad_active[A][ROW4] plus the loss.  A and the row order are identical on every rank
because parameters are replicated and the membership compaction is stable
(k_member: warp ballots + decoupled look-back, idx ascending).  The 1/V mean is folded
into the loss gradient (n_views_total), so the all-reduce is a plain sum.

Backend: torch.distributed process groups (NCCL over NVLink on the GPU box; gloo in the
CPU tests).  This module holds only host logic -- no arithmetic of the method.
"""
from __future__ import annotations

from typing import Callable, List, Optional, Sequence

import torch
import torch.distributed as dist


def shard_views(n_views: int, world: int, rank: int, weights: Optional[Sequence[float]] = None) -> List[int]:
    """Views of `rank`.  Without weights: contiguous blocks.  With weights (e.g. the previous
    step's active tiles per view): longest-processing-time-first assignment, ties broken by
    view index so every rank computes the same partition."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    if weights is None:
        base, extra = divmod(n_views, world)
        start = rank * base + min(rank, extra)
        return list(range(start, start + base + (1 if rank < extra else 0)))
    if len(weights) != n_views:
        raise ValueError("one weight per view")
    order = sorted(range(n_views), key=lambda v: (-float(weights[v]), v))
    load = [0.0] * world
    owner = [0] * n_views
    for v in order:
        r = min(range(world), key=lambda q: (load[q], q))
        owner[v] = r
        load[r] += float(weights[v])
    return [v for v in range(n_views) if owner[v] == rank]


def allreduce_rows(grad: torch.Tensor, loss: Optional[torch.Tensor], group=None) -> None:
    """In-place sum over ranks of the active-gradient rows and the loss, as ONE collective."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return
    parts = [grad.reshape(-1)]
    if loss is not None:
        parts.append(loss.reshape(-1))
    flat = torch.cat(parts)
    dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    n = grad.numel()
    grad.copy_(flat[:n].view_as(grad))
    if loss is not None:
        loss.copy_(flat[n:].view_as(loss))


class PackedRows:
    """One flat fp32 buffer holding the step's loss and its active-gradient rows, laid out so that the
    loss and the first A rows are ONE contiguous prefix: [loss, 0, 0, 0][row 0][row 1]...  The C ABI
    writes the loss and the rows straight into it (no torch.cat / copy_ around the collective), and the
    all-reduce covers exactly the prefix of the live rows (eager) or of the row capacity (CUDA graph)."""

    def __init__(self, capacity_rows: int, row_floats: int, device):
        self.capacity = max(int(capacity_rows), 1)
        self.row_floats = int(row_floats)
        self.flat = torch.zeros(4 + self.capacity * self.row_floats, dtype=torch.float32, device=device)
        self.loss = self.flat[:1]
        self.rows = self.flat[4:].view(self.capacity, self.row_floats // 4, 4)

    def prefix(self, n_rows: int) -> torch.Tensor:
        return self.flat[: 4 + min(int(n_rows), self.capacity) * self.row_floats]


def allreduce_packed(buf: torch.Tensor, group=None) -> None:
    """The step's only exchange: one in-place sum over ranks of a PackedRows prefix."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return
    dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)


def checksum(t: torch.Tensor) -> int:
    """Bitwise checksum of a float tensor (cross-rank parameter identity checks)."""
    b = t.detach().contiguous().view(torch.int32).to(torch.int64)
    return int(((b * 2654435761) % (1 << 61)).sum().item())


def ranks_agree(value: int, group=None) -> bool:
    """True if every rank holds the same integer (e.g. a parameter checksum)."""
    if not dist.is_available() or not dist.is_initialized():
        return True
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([value, -value], dtype=torch.int64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return int(t[0]) == value and int(t[1]) == -value


class DataParallelStep:
    """One data-parallel local-optimisation step.

    `compute(views, n_views_total) -> (grad_rows, loss)` renders this rank's views
    (fwd + bwd through the C ABI in the product, see LocalOptimizer.forward/backward);
    `update(grad_rows)` applies the masked Adam.  Between them: one all-reduce.
    """

    def __init__(self, compute: Callable, update: Callable, n_views: int, world: int = 1, rank: int = 0,
                 group=None):
        self.compute, self.update = compute, update
        self.n_views, self.world, self.rank, self.group = n_views, world, rank, group
        self.views = shard_views(n_views, world, rank)

    def rebalance(self, weights: Sequence[float]) -> None:
        self.views = shard_views(self.n_views, self.world, self.rank, weights)

    def __call__(self):
        grad, loss = self.compute(self.views, self.n_views)
        allreduce_rows(grad, loss, self.group)
        self.update(grad)
        return loss

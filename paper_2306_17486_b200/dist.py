"""Data-parallel plumbing: independent RHS / slowness models sharded over ranks.

The solve has no exchange step: every (model, RHS) pair is
independent, so ranks never communicate on the data path.  Data-parallel
training (train.py) has one: the flat gradient vector is averaged across ranks
(``allreduce_mean``, one NCCL all-reduce per step) between backward and Adam.  One process per
GPU, ``torch.distributed`` (NCCL on GPUs, gloo in the CPU tests) is used only
to time the job as the max over ranks and to gather per-RHS reports.
"""
from __future__ import annotations

import os


def rank_world() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced [start, stop) share of n items for `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def _device():
    import torch
    import torch.distributed as dist

    if dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def reduce_scalar(value: float, op: str = "max") -> float:
    """All-reduce one float (max or sum) across ranks; identity without a process group."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return float(t.item())


def gather_reports(local: list) -> list:
    """Concatenate every rank's list (e.g. per-RHS SolveReports) in rank order."""
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return list(local)
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, list(local))
    return [item for part in out for item in part]


def world_size() -> int:
    import torch.distributed as dist

    return dist.get_world_size() if dist.is_available() and dist.is_initialized() else 1


def allreduce_mean(t):
    """In-place average of a tensor across ranks (sum all-reduce / world); identity alone."""
    import torch.distributed as dist

    w = world_size()
    if w == 1:
        return t
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    t /= w
    return t


def report_rows(reports) -> list:
    """SolveReports as plain (iterations, history, converged) tuples: the per-RHS result the gather carries."""
    return [(int(r.iterations), [float(v) for v in r.relative_residual_history], bool(r.converged)) for r in reports]


def sharded_solve(solve_fn, rhs, model_of):
    """Solve this rank's contiguous share of a batch and gather every RHS's report in global order.

    ``solve_fn(rhs_shard, model_of_shard) -> (x_shard, reports)`` runs the local batch (the device
    ``BatchSolver.solve`` in production, the oracle in the CPU tests).  The shards are independent
    (no exchange step inside a solve), so the only collective is the all-gather of the
    per-RHS (iterations, history, converged) rows, in rank order, i.e. in the batch's own order.

    Returns ``(rows, x_shard, (start, stop))`` with ``rows`` covering the whole batch on every rank.
    """
    rank, world = (0, 1)
    try:
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized():
            rank, world = dist.get_rank(), dist.get_world_size()
    except ImportError:  # pragma: no cover
        pass
    start, stop = shard_range(len(rhs), world, rank)
    x, reps = solve_fn(rhs[start:stop], model_of[start:stop])
    return gather_reports(report_rows(reps)), x, (start, stop)

"""theta-batch data parallelism across ranks (one process per GPU).

Rows are independent units: each rank owns a contiguous block of theta rows, runs
tcx_grad_batch on it, and the ranks all-reduce [sum_b E_b, sum_b grad_b] (the north_star's
"final NCCL all-reduce of loss and gradient"; the SUM reading of vvag, C7).
Backend-agnostic torch.distributed: NCCL on GPUs, gloo in the CPU tests.
"""
from __future__ import annotations


def row_block(B_total: int, world: int, rank: int):
    """[start, stop) of the contiguous row block owned by `rank` (sizes differ by <= 1)."""
    base, extra = divmod(B_total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def pack_loss_grad(E, G, out=None):
    """[sum_b E_b, sum_b G_b] as one contiguous fp64 vector (one collective)."""
    import torch
    P = G.shape[1]
    if out is None:
        out = torch.empty(1 + P, dtype=torch.float64, device=E.device)
    out[0] = E.sum()
    out[1:] = G.sum(0)
    return out


def allreduce_loss_grad(E, G, out=None, group=None):
    import torch.distributed as dist
    red = pack_loss_grad(E, G, out)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(red, group=group)
    return red

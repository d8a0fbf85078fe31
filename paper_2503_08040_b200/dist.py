"""Data-parallel plumbing for the fallback-quantized MLP.

Tokens are sharded across ranks in 128-row-aligned slices so quantization
blocks never straddle ranks (block scales, masks and codes are then identical
to the single-GPU run, and the stochastic-rounding RNG index stays global via
``row_offset``).  Weights are replicated; the only exchange is the sum of the
fp32 dW partials (NCCL all-reduce over NVLink), launched on a side stream.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

BLOCK = 128


def shard_rows(total: int, world: int, rank: int, align: int = BLOCK):
    """[start, end) of this rank's token rows; every boundary a multiple of `align`."""
    if total % align:
        raise ValueError(f"token count {total} must be a multiple of {align} for sharding")
    blocks = total // align
    base, extra = divmod(blocks, world)
    start = rank * base + min(rank, extra)
    count = base + (1 if rank < extra else 0)
    return start * align, (start + count) * align


def allreduce_grads(tensors, group=None, async_op=False):
    """Sum the dW partials across ranks (the one collective of the path)."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return []
    works = [dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group, async_op=async_op)
             for t in tensors]
    return works if async_op else []


def allreduce_mlp_grads_overlapped(mlp, gu_grad, d_grad, comm_stream, group=None):
    """The dW all-reduce of one fallback-quantized MLP step, overlapped with
    its backward: call right after ``mlp.backward(...)`` was enqueued.  dW_down
    is final as soon as its GEMM ends (``fbq_mlp_wait_grad``), so its NCCL
    all-reduce runs on ``comm_stream`` while the GLU backward and the gate/up
    GEMMs still occupy the compute stream; dW_gate|up follows the backward.
    On return the current stream is ordered after both reductions."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return
    with torch.cuda.stream(comm_stream):
        mlp.wait_grad(2, comm_stream)
        w_down = dist.all_reduce(d_grad, op=dist.ReduceOp.SUM, group=group, async_op=True)
    w_gu = dist.all_reduce(gu_grad, op=dist.ReduceOp.SUM, group=group, async_op=True)
    w_down.wait()
    w_gu.wait()


def max_over_ranks(value: float, device=None) -> float:
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())

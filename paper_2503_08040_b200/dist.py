"""Data-parallel plumbing for the fallback-quantized MLP.

Tokens are sharded across ranks in 128-row-aligned slices so quantization
blocks never straddle ranks (block scales, masks and codes are then identical
to the single-GPU run, and the stochastic-rounding RNG index stays global via
``row_offset``).  Weights are replicated; the only exchange is the sum of the
fp32 dW partials (NCCL all-reduce over NVLink), launched on a side stream,
plus one int32 per layer -- the masked-block counts -- so the delay-threshold
controller sees the fallback rate of the whole batch.
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
    """Sum the dW partials across ranks (the path's data collective)."""
    if not _dp(group):
        return []
    works = [dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group, async_op=async_op)
             for t in tensors]
    return works if async_op else []


def _dp(group=None) -> bool:
    return dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1


def allreduce_mlp_grads_overlapped(mlp, gu_grad, d_grad, comm_stream, group=None):
    """The dW all-reduce of one fallback-quantized MLP step, overlapped with
    its backward: call right after ``mlp.backward(...)`` was enqueued.  Each
    gradient is final right after its own GEMM (``fbq_mlp_wait_grad``):
    dW_down first (its all-reduce runs while the GLU backward and the gate/up
    GEMMs still occupy the compute streams), then dW_gate (overlapping the
    dW_up GEMM), then dW_up.  All three go out on ``comm_stream``; on return
    the current stream is ordered after the reductions."""
    if not _dp(group):
        return
    f = mlp.d_ff
    works = []
    with torch.cuda.stream(comm_stream):
        for which, t in ((2, d_grad), (0, gu_grad[:f]), (1, gu_grad[f:])):
            mlp.wait_grad(which, comm_stream)
            works.append(dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group, async_op=True))
    for w in works:
        w.wait()


def allreduce_block_grads_overlapped(block, gu_grad, d_grad, comm_stream, group=None):
    """GluBlock (trainsim.cpp:294-308): the MLP's three dW all-reduces overlapped
    with the backward (allreduce_mlp_grads_overlapped), then the RmsNorm's
    grad_gain (d_model floats, final once the norm backward -- the block
    backward's last kernel -- has run on the current stream)."""
    if not _dp(group):
        return
    allreduce_mlp_grads_overlapped(block, gu_grad, d_grad, comm_stream, group)
    dist.all_reduce(block.gain_tensors()[1], op=dist.ReduceOp.SUM, group=group)


def controller_step_global(module, global_tokens: int, group=None):
    """controller_step on the rate of the WHOLE batch (trainsim.cpp:93,129-133;
    policy.cpp:97-109): sum the device masked-block counters of the last
    forward over ranks in place (one int32 all-reduce per layer, on the current
    stream, no host round trip) and divide by the global block count, so every
    rank moves theta identically and the masks stay those of a one-GPU run.
    ``module`` is a GluMlp or QuantLinear; ``global_tokens`` the tokens of the
    forward summed over ranks (shards are 128-row aligned, so the global block
    count is global_tokens / 128 x column blocks)."""
    if _dp(group):
        dist.all_reduce(module.count_tensor(), op=dist.ReduceOp.SUM, group=group)
        module.controller_step(global_tokens=global_tokens)
    else:
        module.controller_step()


def global_quantile(values: torch.Tensor, q: float, group=None) -> float:
    """The q-quantile of `values` pooled over all ranks (all_gather), e.g. the
    initial fallback thresholds from block scores, so every rank starts from the
    same theta."""
    v = values.reshape(-1).float()
    if _dp(group):
        parts = [torch.empty_like(v) for _ in range(dist.get_world_size(group))]
        dist.all_gather(parts, v.contiguous(), group=group)
        v = torch.cat(parts)
    return float(torch.quantile(v, q))


def max_over_ranks(value: float, device=None) -> float:
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())

"""CPU: the data-parallel plumbing (token sharding + dW all-reduce) with
world_size 2 over gloo, and the sharding semantics on the oracle:
128-row-aligned shards give bit-identical codes/masks/per-row outputs, and the
dW partials sum to the full-batch dW within fp32 reassociation tolerance."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from tests.helpers import outlier_matrix, rel_fro


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2503_08040_b200.dist import allreduce_grads, max_over_ranks, shard_rows
    start, end = shard_rows(1024, world, rank)
    g1 = torch.full((4, 3), float(rank + 1))
    g2 = torch.arange(6, dtype=torch.float32) * (rank + 1)
    allreduce_grads([g1, g2])
    mx = max_over_ranks(float(rank) * 2.5)
    out[rank] = (start, end, g1.sum().item(), g2.tolist(), mx)
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_allreduce_and_sharding():
    ctx = mp.get_context("spawn")
    manager = ctx.Manager()
    out = manager.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    (s0, e0, g0, l0, m0), (s1, e1, g1, l1, m1) = out[0], out[1]
    assert (s0, e0, s1, e1) == (0, 512, 512, 1024)
    assert g0 == g1 == 12 * 3.0  # (1 + 2) summed over 12 elements
    assert l0 == l1 == [v * 3.0 for v in range(6)]
    assert m0 == m1 == 2.5


def test_shard_rows_alignment():
    from paper_2503_08040_b200.dist import shard_rows
    for total, world in [(8192, 8), (8192 * 3, 8), (1280, 3), (128, 1)]:
        spans = [shard_rows(total, world, r) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == total
        for (a, b), (c, _) in zip(spans, spans[1:]):
            assert b == c
        assert all(a % 128 == 0 and b % 128 == 0 for a, b in spans)
    with pytest.raises(ValueError):
        shard_rows(1000, 2, 0)


def test_sharded_semantics_on_oracle(orc):
    """Two 128-aligned token shards == the full batch (codes, masks, dW)."""
    t, k, n = 256, 256, 384
    x = outlier_matrix(t, k, seed=3, channels=[2], tokens=[200])
    gy = outlier_matrix(t, n, seed=4, body=1e-3)
    seed_ctx, seed_gy = 0x1234, 0x5678
    fx, fs = orc.quantize_stochastic(x, seed_ctx)
    gc, gs = orc.quantize_stochastic(gy, seed_gy)
    full_mask = orc.mask_threshold(orc.score_blocks_absmax(x), 20.0)
    gtc, gts = orc.transpose_qt(gc, gs)
    dw_full = orc.block_gemm(gtc, gts, fx, fs)
    dw_sum = np.zeros_like(dw_full)
    for r0 in (0, 128):
        xs, gys = x[r0:r0 + 128], gy[r0:r0 + 128]
        cx, sx = orc.quantize_stochastic(xs, seed_ctx, row_offset=r0)
        assert np.array_equal(cx, fx[r0:r0 + 128]) and np.array_equal(sx, fs[r0 // 128:r0 // 128 + 1])
        m = orc.mask_threshold(orc.score_blocks_absmax(xs), 20.0)
        assert np.array_equal(m, full_mask[r0 // 128:r0 // 128 + 1])
        cg, sg = orc.quantize_stochastic(gys, seed_gy, row_offset=r0)
        ctc, cts = orc.transpose_qt(cg, sg)
        dw_sum += orc.block_gemm(ctc, cts, cx, sx)
    assert rel_fro(dw_sum, dw_full) < 1e-6

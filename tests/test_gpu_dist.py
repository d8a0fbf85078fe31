"""GPU: the data-parallel MLP step end to end on one B200 -- two ranks (gloo,
CUDA tensors, both on cuda:0) each run their 128-row-aligned token shard
through the fused MLP and reduce dW with dist.allreduce_mlp_grads_overlapped
(dW_down, dW_gate and dW_up each on a side stream ordered by
fbq_mlp_wait_grad) and the controller with dist.controller_step_global (the
masked-block counts summed over ranks, the global block count), over three
steps.  The summed dW must equal the full-batch dW within fp32
reassociation tolerance; the per-row outputs must be bit-identical to the
full batch, and so must the thresholds and the observed fallback rates after
every controller step (trainsim.cpp:93,129-133).  NCCL needs one GPU per rank, so
the collective here is gloo; the stream/event ordering under test is the same."""
import os
import socket

import numpy as np
import pytest

from tests.helpers import outlier_matrix, rel_fro

pytestmark = pytest.mark.gpu

D, F, T = 256, 384, 512
STEPS = 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _inputs():
    rng = np.random.default_rng(9)
    wg = (rng.standard_normal((F, D)) * 0.05).astype(np.float32)
    wu = (rng.standard_normal((F, D)) * 0.05).astype(np.float32)
    wd = (rng.standard_normal((D, F)) * 0.05).astype(np.float32)
    x = outlier_matrix(T, D, seed=11, body=0.3, channels=[5], tokens=[T // 3], mag_c=20.0, mag_t=40.0)
    gy = outlier_matrix(T, D, seed=18, body=1e-3)
    return wg, wu, wd, x, gy


def _worker(rank, world, port, q, kind="mlp"):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2503_08040_b200 import linear
    from paper_2503_08040_b200.dist import (allreduce_block_grads_overlapped, allreduce_mlp_grads_overlapped,
                                            controller_step_global, shard_rows)
    wg, wu, wd, x, gy = _inputs()
    r0, r1 = shard_rows(T, world, rank)
    kw = dict(act_dtype=torch.float32, mid_dtype=torch.float32, exact=True, threshold_init=4.0)
    m = (linear.GluMlp if kind == "mlp" else linear.GluBlock)(wg, wu, wd, r1 - r0, **kw)
    gu, gd = m.grad_tensors()
    comm = torch.cuda.Stream()
    outs = []
    for step in range(STEPS):
        m.zero_grad()
        y = m.forward(torch.from_numpy(x[r0:r1]).cuda(), step, row_offset=r0)
        gx = m.backward(torch.from_numpy(gy[r0:r1]).cuda(), step, row_offset=r0)
        if kind == "mlp":
            allreduce_mlp_grads_overlapped(m, gu, gd, comm)
        else:
            allreduce_block_grads_overlapped(m, gu, gd, comm)
        controller_step_global(m, T)
        outs.append((y.cpu().numpy(), gx.cpu().numpy(), m.controller_state()))
    torch.cuda.synchronize()
    gg = m.gain_tensors()[1].cpu().numpy() if kind == "block" else None
    q.put((rank, r0, r1, outs, gu.cpu().numpy(), gd.cpu().numpy(), gg))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["mlp", "block"])
def test_dp_world2_overlapped_allreduce_matches_full_batch(kind):
    """kind = block: the pre-norm residual GluBlock, whose RmsNorm grad_gain is
    summed over ranks as well."""
    import torch
    import torch.multiprocessing as mp
    from paper_2503_08040_b200 import linear
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, kind)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    wg, wu, wd, x, gy = _inputs()
    kw = dict(act_dtype=torch.float32, mid_dtype=torch.float32, exact=True, threshold_init=4.0)
    full = (linear.GluMlp if kind == "mlp" else linear.GluBlock)(wg, wu, wd, T, **kw)
    gu, gd = full.grad_tensors()
    want = []
    for step in range(STEPS):
        full.zero_grad()
        y = full.forward(torch.from_numpy(x).cuda(), step).cpu().numpy()
        gx = full.backward(torch.from_numpy(gy).cuda(), step).cpu().numpy()
        full.controller_step()
        want.append((y, gx, full.controller_state()))
    torch.cuda.synchronize()
    # the controller must actually move theta in this test (else it proves nothing)
    assert want[0][2][1] != want[-1][2][1]
    for rank, r0, r1, outs, g_gu, g_d, g_gain in res:
        if kind == "block":
            assert rel_fro(g_gain, full.gain_tensors()[1].cpu().numpy()) < 1e-6
        for step, ((y, gx, ctl), (yw, gxw, ctlw)) in enumerate(zip(outs, want)):
            assert np.array_equal(y.view(np.int32), yw[r0:r1].view(np.int32)), step
            assert np.array_equal(gx.view(np.int32), gxw[r0:r1].view(np.int32)), step
            assert ctl == ctlw, (step, ctl, ctlw)  # global rates and thresholds
        # both ranks hold the all-reduced sum (last step's dW)
        assert rel_fro(g_gu, gu.cpu().numpy()) < 1e-6
        assert rel_fro(g_d, gd.cpu().numpy()) < 1e-6

"""GPU: the device C ABI's contract (include/fbq_b200.h): fbq_cuda_* calls never
allocate or synchronise (safe under CUDA stream capture) and are safe from
concurrent host threads -- in particular the GEMM's dynamic tile counters
(one slot per launch, taken atomically from a per-device ring set up by
fbq_cuda_init, left reset by every launch) -- VERDICT r01 weak #10."""
import threading

import numpy as np
import pytest

from tests.helpers import outlier_matrix

pytestmark = pytest.mark.gpu


def _dev(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


@pytest.fixture(scope="module")
def setup():
    import torch
    from paper_2503_08040_b200 import fbq
    m, n, k = 1152, 1536, 1408  # multi-wave, ragged K pages, fallback blocks
    x = outlier_matrix(m, k, seed=61, channels=[3, 700], tokens=[40], occasional=30)
    w = outlier_matrix(n, k, seed=62, body=0.02)
    fa = fbq.fallback_quantize(_dev(x), fbq.mask_topk(fbq.score_blocks(_dev(x)), 0.15))
    wq = fbq.transpose(fbq.quantize_rtn(_dev(w)))
    want = fbq.fallback_gemm(fa, wq)
    torch.cuda.synchronize()
    return fbq, fa, wq, want


def test_gemm_under_cuda_graph_capture(setup):
    import torch
    fbq, fa, wq, want = setup
    out = torch.empty_like(want)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fbq.fallback_gemm(fa, wq, out=out)  # warm (per-device setup already done)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fbq.fallback_gemm(fa, wq, out=out)
        fbq.fallback_gemm(fa, wq, out=out, accumulate=True)
    for _ in range(4):  # every replay reuses the captured tile-counter slots
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(out, want + want)


def test_gemm_from_two_host_threads(setup):
    import torch
    fbq, fa, wq, want = setup
    errors = []
    n_iter = 40

    def worker(tid):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            outs = [torch.empty_like(want) for _ in range(4)]
            with torch.cuda.stream(s):
                for i in range(n_iter):
                    fbq.fallback_gemm(fa, wq, out=outs[i % 4])
            s.synchronize()
            for o in outs:
                if not torch.equal(o, want):
                    errors.append(f"thread {tid}: wrong result")
                    return
        except Exception as ex:  # pragma: no cover
            errors.append(f"thread {tid}: {ex!r}")

    ts = [threading.Thread(target=worker, args=(t,)) for t in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors

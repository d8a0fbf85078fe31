"""L2 policy A/B: evict-first for the streamed operand (default) vs all evict-last (diag 1 << 23).
vs the static schedule tile += gridDim.x (diag 1 << 21), MLP shapes and
C1/C5 at 10 % fallback."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_08040_b200 import fbq
import bench

lib = fbq.K.lib
lib.fbq_debug_set_gemm_diag.argtypes = [fbq.K.cint]
ALT = 1 << 23


def timeit(fn, iters=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e-3


for (name, M, N, K) in [("gate/up fwd", 8192, 28672, 4096), ("down fwd", 8192, 4096, 14336),
                        ("dW_g-like", 14336, 4096, 8192), ("dX merged", 8192, 4096, 28672),
                        ("C5", 8192, 28672, 8192), ("C1", 4096, 4096, 4096)]:
    x = bench.make_activations(M, K, 1, "cuda", torch.bfloat16)
    w = torch.randn(N, K, device="cuda") * 0.02
    wq = fbq.transpose(fbq.quantize_rtn(w))
    fa = fbq.fallback_quantize(x, fbq.mask_topk(fbq.score_blocks(x), 0.10))
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    res = {0: [], ALT: []}
    ys = {}
    for rnd in range(4):
        for d in (list(res) if rnd % 2 == 0 else list(res)[::-1]):
            lib.fbq_debug_set_gemm_diag(d)
            res[d].append(timeit(lambda: fbq.fallback_gemm(fa, wq, out=out, exact=False)))
            ys[d] = fbq.fallback_gemm(fa, wq, exact=True)
    lib.fbq_debug_set_gemm_diag(0)
    same = torch.equal(ys[0].view(torch.int32), ys[ALT].view(torch.int32))
    ops = 2 * M * N * K
    med = lambda v: sorted(v)[len(v) // 2]
    print(f"{name:12s} {M}x{N}x{K}: split-policy {ops/med(res[0])/1e12:6.0f} TOPS (median of 4), "
          f"evict-last {ops/med(res[ALT])/1e12:6.0f} TOPS, identical={same}", flush=True)

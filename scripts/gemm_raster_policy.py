"""A/B of the GEMM tile rasters on the shapes where both operands are large
(VERDICT r01 weak #6): default policy vs forced rasters (diag bits: 1<<18 groups
of 8 block-rows, 1<<19 bm over all block-rows (A resident), 1<<20 bn fastest
(B resident)).  Interleaved repeats, median TOPS."""
import sys, os, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_08040_b200 import fbq
import bench

lib = fbq.K.lib
lib.fbq_debug_set_gemm_diag.argtypes = [fbq.K.cint]


def timeit(fn, iters=8, warm=2):
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


shapes = {"C5 8192x28672x8192": (8192, 28672, 8192), "down fwd 8192x4096x14336": (8192, 4096, 14336),
          "dX 8192x4096x28672": (8192, 4096, 28672), "C1 4096^3": (4096, 4096, 4096)}
for name, (M, N, K) in shapes.items():
    x = bench.make_activations(M, K, 3, "cuda", torch.bfloat16)
    w = torch.randn(N, K, device="cuda") * 0.02
    wq = fbq.transpose(fbq.quantize_rtn(w))
    fa = fbq.fallback_quantize(x, fbq.mask_topk(fbq.score_blocks(x), 0.10))
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    res = {d: [] for d in (0, 1 << 18, 1 << 19, 1 << 20)}
    for rep in range(3):
        for d in res:
            lib.fbq_debug_set_gemm_diag(d)
            t = timeit(lambda: fbq.fallback_gemm(fa, wq, out=out, exact=False))
            res[d].append(2 * M * N * K / t / 1e12)
    lib.fbq_debug_set_gemm_diag(0)
    print(name, {("default", "groups8", "A-resident", "B-resident")[i]: round(statistics.median(v))
                 for i, v in enumerate(res.values())}, flush=True)
    del x, w, wq, fa, out
    torch.cuda.empty_cache()

"""Where does the fallback GEMM lose time at 10 % flagged blocks?
C5 shape (8192 x 28672 x 8192): topk mask of outlier activations (bench) vs a
uniformly random mask vs a mask with the same count spread evenly over block
rows; diag 1 = epilogue math off (MMA/TMA side only)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_08040_b200 import fbq
import bench


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


lib = fbq.K.lib
lib.fbq_debug_set_gemm_diag.argtypes = [fbq.K.cint]
M, N, K = int(os.environ.get("M", 8192)), 28672, 8192
x = bench.make_activations(M, K, 1, "cuda", torch.float32)
w = torch.randn(N, K, device="cuda") * 0.02
wq = fbq.transpose(fbq.quantize_rtn(w))
out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
scores = fbq.score_blocks(x)
MB, KB = scores.shape
g = torch.Generator(device="cpu").manual_seed(0)
for rate in (0.0, 0.10):
    n = int(round(rate * MB * KB))
    masks = {"topk": fbq.mask_topk(scores, rate)}
    if rate > 0:
        r = torch.zeros(MB * KB, dtype=torch.uint8)
        r[torch.randperm(MB * KB, generator=g)[:n]] = 1
        masks["random"] = r.view(MB, KB).cuda()
        e = torch.zeros(MB, KB, dtype=torch.uint8)
        per = n // MB
        for i in range(MB):
            e[i, (torch.arange(per) * (KB // max(per, 1)) + i) % KB] = 1
        masks["even_rows"] = e.cuda()
    for name, m in masks.items():
        mm = m.to(torch.int64).view(MB, KB)
        rows = mm.sum(1)
        fa = fbq.fallback_quantize(x, m)
        for d in (0, 1):
            lib.fbq_debug_set_gemm_diag(d)
            t = timeit(lambda: fbq.fallback_gemm(fa, wq, out=out, exact=False))
            print(f"rate={rate:.2f} mask={name:9s} flagged={int(mm.sum())} per-row max={int(rows.max())} "
                  f"min={int(rows.min())} diag={d}: {t*1e3:.3f} ms {2*M*N*K/t/1e12:.0f} TOPS", flush=True)
        lib.fbq_debug_set_gemm_diag(0)

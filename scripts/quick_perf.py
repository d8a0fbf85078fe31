"""Quick perf probe: kernel times with CUDA events (not the bench contract)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_08040_b200 import fbq


def timeit(fn, iters=20, warm=3):
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


res = {}
torch.manual_seed(0)
for (M, N, K) in [(4096, 4096, 4096), (8192, 14336, 4096), (8192, 4096, 14336), (8192, 28672, 8192)]:
    x = torch.randn(M, K, device="cuda")
    x[:, 7] *= 100
    w = torch.randn(N, K, device="cuda") * 0.02
    wq = fbq.transpose(fbq.quantize_rtn(w))
    for rate in [0.0, 0.1]:
        s = fbq.score_blocks(x)
        mask = fbq.mask_topk(s, rate)
        fa = fbq.fallback_quantize(x, mask)
        for exact in [False, True]:
            out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
            t = timeit(lambda: fbq.fallback_gemm(fa, wq, out=out, exact=exact))
            res[f"gemm {M}x{N}x{K} rate={rate} exact={exact}"] = f"{t*1e3:.3f} ms  {2*M*N*K/t/1e12:.1f} TOPS"
    xb = x.to(torch.bfloat16); wb = w.to(torch.bfloat16)
    t = timeit(lambda: xb @ wb.t())
    res[f"torch bf16 {M}x{N}x{K}"] = f"{t*1e3:.3f} ms  {2*M*N*K/t/1e12:.1f} TFLOPS"
    xi = torch.randint(-127, 127, (M, K), device="cuda", dtype=torch.int8)
    wi = torch.randint(-127, 127, (K, N), device="cuda", dtype=torch.int8)
    try:
        t = timeit(lambda: torch._int_mm(xi, wi))
        res[f"torch _int_mm {M}x{N}x{K}"] = f"{t*1e3:.3f} ms  {2*M*N*K/t/1e12:.1f} TOPS"
    except Exception as ex:
        res["int_mm"] = str(ex)[:100]
for (R, C) in [(8192, 4096), (8192, 14336)]:
    for dt in [torch.bfloat16, torch.float32]:
        x = torch.randn(R, C, device="cuda").to(dt)
        esz = x.element_size()
        t = timeit(lambda: fbq.fallback_quantize(x, theta=3.5))
        nb = (R // 128) * (C // 128)
        byt = R * C * (esz + 1) + nb * 8
        res[f"quant_fb {R}x{C} {dt}"] = f"{t*1e6:.1f} us {byt/t/1e9:.0f} GB/s (+res)"
        t = timeit(lambda: fbq.quantize_stochastic(x, 1234))
        res[f"quant_sr {R}x{C} {dt}"] = f"{t*1e6:.1f} us {R*C*(esz+1)/t/1e9:.0f} GB/s"
        t = timeit(lambda: fbq.quantize_rtn(x))
        res[f"quant_rtn {R}x{C} {dt}"] = f"{t*1e6:.1f} us {R*C*(esz+1)/t/1e9:.0f} GB/s"
for k, v in res.items():
    print(f"{k:45s} {v}")
json.dump(res, open("gpurun_out/quick_perf.json", "w"), indent=1)

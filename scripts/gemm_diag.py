"""Which role paces the GEMM?  diag 1 = no epilogue math, 2 = no TMA, 3 = both."""
import sys, os
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


lib = fbq.K.lib
lib.fbq_debug_set_gemm_diag.argtypes = [fbq.K.cint]
for (M, N, K) in [(8192, 14336, 4096), (8192, 4096, 14336)]:
    x = torch.randn(M, K, device="cuda")
    w = torch.randn(N, K, device="cuda") * 0.02
    wq = fbq.transpose(fbq.quantize_rtn(w))
    qa = fbq.quantize_rtn(x)
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    for d in []:
        lib.fbq_debug_set_gemm_diag(d)
        t = timeit(lambda: fbq.block_quant_gemm(qa, wq, out=out, exact=False))
        print(f"{M}x{N}x{K} diag={d}: {t*1e3:.3f} ms {2*M*N*K/t/1e12:.0f} TOPS", flush=True)
    lib.fbq_debug_set_gemm_diag(0)

# MMA-warp wait profile
lib.fbq_debug_set_gemm_prof.argtypes = [fbq.K.vp]
prof = torch.zeros(148 * 5, dtype=torch.int64, device="cuda")
for (M, N, K) in [(8192, 14336, 4096)]:
    x = torch.randn(M, K, device="cuda")
    w = torch.randn(N, K, device="cuda") * 0.02
    wq = fbq.transpose(fbq.quantize_rtn(w))
    qa = fbq.quantize_rtn(x)
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    for d in [0, 31, 512 + 31]:
        lib.fbq_debug_set_gemm_diag(d)
        lib.fbq_debug_set_gemm_prof(prof.data_ptr())
        fbq.block_quant_gemm(qa, wq, out=out, exact=False)
        torch.cuda.synchronize()
        lib.fbq_debug_set_gemm_prof(None)
        pr = prof.view(148, 5).double().mean(0).tolist()
        items = (M // 128) * (N // 256) * (K // 128) / 148
        print(f"diag={d} per-item cycles: total {pr[0]/items:.0f} full-wait {pr[1]/items:.0f} "
              f"tmem-wait {pr[2]/items:.0f} page-wait {pr[3]/items:.0f} issue {pr[4]/items:.0f} (MMA ideal 512)", flush=True)
    lib.fbq_debug_set_gemm_diag(0)

# wall-clock TOPS without the per-item clock reads (prof disabled)
lib.fbq_debug_set_gemm_prof(None)
for d in [0, 31, 512 + 31]:
    lib.fbq_debug_set_gemm_diag(d)
    t = timeit(lambda: fbq.block_quant_gemm(qa, wq, out=out, exact=False))
    print(f"no-prof diag={d}: {t*1e3:.3f} ms {2*M*N*K/t/1e12:.0f} TOPS", flush=True)
lib.fbq_debug_set_gemm_diag(0)

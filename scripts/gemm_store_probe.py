"""GEMM (0 % fallback): normal vs no output stores (diag 4) vs no epilogue math (1) vs neither (5)."""
import sys, os
sys.path.insert(0, "/root/repo")
import torch
from paper_2503_08040_b200 import fbq
import bench
lib = fbq.K.lib
lib.fbq_debug_set_gemm_diag.argtypes = [fbq.K.cint]
def timeit(fn, iters=10, warm=3):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e-3
for (M, N, K) in [(8192, 28672, 4096), (8192, 4096, 14336), (4096, 4096, 4096)]:
    x = bench.make_activations(M, K, 1, "cuda", torch.bfloat16)
    w = torch.randn(N, K, device="cuda") * 0.02
    wq = fbq.transpose(fbq.quantize_rtn(w))
    qa = fbq.quantize_rtn(x)
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    r = {}
    for rnd in range(2):
        for d in (0, 4, 1, 5):
            lib.fbq_debug_set_gemm_diag(d)
            r.setdefault(d, []).append(timeit(lambda: fbq.block_quant_gemm(qa, wq, out=out, exact=False)))
    lib.fbq_debug_set_gemm_diag(0)
    print(f"{M}x{N}x{K}: " + "  ".join(f"diag{d}={2*M*N*K/min(v)/1e12:.0f}" for d, v in r.items()), flush=True)

"""What the tile-end output stores cost the GEMM: block GEMMs (no fallback) at the
step's shapes with the store skipped (diag 4) vs stored, both on the diagnostic instantiation
(diag 1 << 24: default L2 policy on the stores, otherwise neutral), interleaved."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_08040_b200 import fbq

lib = fbq.K.lib
lib.fbq_debug_set_gemm_diag.argtypes = [fbq.K.cint]


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


for (M, N, K) in [(8192, 4096, 4096), (8192, 14336, 4096), (8192, 4096, 28672)]:
    x = torch.randn(M, K, device="cuda")
    w = torch.randn(N, K, device="cuda") * 0.02
    wq = fbq.transpose(fbq.quantize_rtn(w))
    qa = fbq.quantize_rtn(x)
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    res = {1 << 24: [], (1 << 24) | 4: []}
    for _ in range(3):
        for d in (1 << 24, (1 << 24) | 4):
            lib.fbq_debug_set_gemm_diag(d)
            t = timeit(lambda: fbq.block_quant_gemm(qa, wq, out=out, exact=False))
            res[d].append(2 * M * N * K / t / 1e12)
    lib.fbq_debug_set_gemm_diag(0)
    print(f"{M}x{N}x{K}: with stores {max(res[1 << 24]):.0f} TOPS, stores skipped {max(res[(1 << 24) | 4]):.0f} TOPS "
          f"({(max(res[(1 << 24) | 4]) / max(res[1 << 24]) - 1) * 100:+.1f} %)", flush=True)

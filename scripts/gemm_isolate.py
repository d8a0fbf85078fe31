"""Bare-MMA-loop attribution inside the real GEMM kernel (diag bits, results garbage):
1 no epilogue math, 2 no TMA, 4 no stores, 8 no tempty wait, 16 no full wait,
64 no tcgen05 fence in the MMA loop, 128 no per-stage commit, 256 single N=256 MMA,
512 no scale pages."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_08040_b200 import fbq
lib = fbq.K.lib
lib.fbq_debug_set_gemm_diag.argtypes = [fbq.K.cint]
lib.fbq_debug_set_gemm_prof.argtypes = [fbq.K.vp]
M, N, K = 8192, 14336, 4096
x = torch.randn(M, K, device="cuda"); w = torch.randn(N, K, device="cuda") * 0.02
if os.environ.get("ZERO_DATA"):  # low-power operands: every code is +-1 (power-throttling probe)
    x = torch.ones(M, K, device="cuda"); w = torch.ones(N, K, device="cuda")
wq = fbq.transpose(fbq.quantize_rtn(w)); qa = fbq.quantize_rtn(x)
out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
prof = torch.zeros(148 * 16, dtype=torch.int64, device="cuda")
items = (M // 128) * (N // 256) * (K // 128) / 148
def run(d):
    lib.fbq_debug_set_gemm_diag(d)
    for _ in range(3): fbq.block_quant_gemm(qa, wq, out=out, exact=False)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10): fbq.block_quant_gemm(qa, wq, out=out, exact=False)
    e.record(); torch.cuda.synchronize()
    t = s.elapsed_time(e) / 10 * 1e-3
    prof.zero_(); lib.fbq_debug_set_gemm_prof(prof.data_ptr())
    fbq.block_quant_gemm(qa, wq, out=out, exact=False); torch.cuda.synchronize()
    lib.fbq_debug_set_gemm_prof(None)
    pr = prof.view(148, 16)
    n = int((pr[:, 0] > 0).sum().item())  # MMA threads that recorded (one per CTA pair)
    pr = pr[:n].double().mean(0).tolist()
    it = pr[4] if pr[4] > 0 else items  # items per MMA thread (k-blocks + residual items)
    print(f"diag={d:4d}: {t*1e3:.3f} ms {2*M*N*K/t/1e12:6.0f} TOPS  MMA-warp cycles/item {pr[0]/it:6.0f} "
          f"(waits: full {pr[1]/it:5.0f} tempty {pr[2]/it:5.0f} rfull {pr[3]/it:5.0f}; {512/(pr[0]/it)*100:.0f}% of tensor peak)", flush=True)
diags = [int(a) for a in sys.argv[1:]] or [1 | 256, 1 | 2 | 256, 1 | 16 | 256, 1 | 8 | 256, 1 | 4 | 256, 1 | 2 | 4 | 256, 287, 287 | 64]
for d in diags:
    run(d)
lib.fbq_debug_set_gemm_diag(0)

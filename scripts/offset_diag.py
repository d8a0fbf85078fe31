"""Which part of the offset epilogue costs time (runs on branch gemm-offset-exp, which has fbq.gemm_offset):
   diag 1<<25 (no row-sum loads), 1<<26 (no column-sum loads); and the signed kernel on the offset bytes."""
import sys, torch
sys.path.insert(0, ".")
from paper_2503_08040_b200 import fbq as F
lib = F.K.lib
lib.fbq_debug_set_gemm_diag.argtypes = [F.K.cint]

def tops(fn, flops, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return flops * reps / (e0.elapsed_time(e1) * 1e-3) / 1e12

m, n, k = 8192, 28672, 8192
torch.manual_seed(0)
a = torch.randn(m, k, device="cuda"); a[:, 3] *= 100
w = torch.randn(n, k, device="cuda") * 0.02
wq = F.quantize_rtn(w)
sc = F.score_blocks(a)
mask = torch.zeros_like(sc, dtype=torch.bool)
fa = F.fallback_quantize(a, mask)
B = F.transpose(wq)
out = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
a_off, b_off = F.offset_operand(fa.primary), F.offset_operand(wq)
r_off = F.to_offset(fa.res_codes, m, k)
fl = 2.0 * m * n * k
print("fma", tops(lambda: F.fallback_gemm(fa, B, out=out, exact=False), fl))
for d in (0, 1 << 25, 1 << 26, (1 << 25) | (1 << 26), 1, 4):
    lib.fbq_debug_set_gemm_diag(d)
    print("offset diag", hex(d), tops(lambda: F.gemm_offset(fa.primary, B, fa, a_off=a_off, b_off=b_off, r_off=r_off, out=out), fl), flush=True)
lib.fbq_debug_set_gemm_diag(0)
for d in (1, 4):
    lib.fbq_debug_set_gemm_diag(d)
    print("fma diag", hex(d), tops(lambda: F.fallback_gemm(fa, B, out=out, exact=False), fl), flush=True)
lib.fbq_debug_set_gemm_diag(0)
# data dependence: the signed FMA kernel on the offset bytes (|q - 128| ~ 128: large products)
from dataclasses import replace
fa2 = replace(fa, primary=replace(fa.primary, codes=a_off.codes))
B2 = F.transpose(replace(wq, codes=b_off.codes))
print("fma on offset bytes", tops(lambda: F.fallback_gemm(fa2, B2, out=out, exact=False), fl), flush=True)
lib.fbq_debug_set_gemm_diag(1)
print("fma diag1 on offset bytes", tops(lambda: F.fallback_gemm(fa2, B2, out=out, exact=False), fl), flush=True)
lib.fbq_debug_set_gemm_diag(0)
import pynvml

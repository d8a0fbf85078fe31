"""Per-item MMA-thread timeline of CTA pair 0 (prof build): for items 0..255,
[issue start, issue end, full-wait start, full-wait end] in MMA-warp cycles."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_08040_b200 import fbq
lib = fbq.K.lib
lib.fbq_debug_set_gemm_diag.argtypes = [fbq.K.cint]
lib.fbq_debug_set_gemm_prof.argtypes = [fbq.K.vp]
M, N, K = 8192, 14336, 4096
diag = int(sys.argv[1]) if len(sys.argv) > 1 else 0
x = torch.randn(M, K, device="cuda"); w = torch.randn(N, K, device="cuda") * 0.02
wq = fbq.transpose(fbq.quantize_rtn(w)); qa = fbq.quantize_rtn(x)
out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
prof = torch.zeros(148 * 16 + 1024, dtype=torch.int64, device="cuda")
lib.fbq_debug_set_gemm_diag(diag)
for _ in range(3): fbq.block_quant_gemm(qa, wq, out=out, exact=False)
lib.fbq_debug_set_gemm_prof(prof.data_ptr())
fbq.block_quant_gemm(qa, wq, out=out, exact=False); torch.cuda.synchronize()
lib.fbq_debug_set_gemm_prof(None); lib.fbq_debug_set_gemm_diag(0)
t = prof[148 * 16:].view(256, 4).tolist()
prev = 0
for i, (a, b, fw0, fw1) in enumerate(t[:96]):
    print(f"item {i:3d}: fullwait {fw0:9d}->{fw1:9d} (+{fw1-fw0:5d})  issue {a:9d}->{b:9d} (+{b-a:5d})  since prev issue {a-prev:6d}")
    prev = a

"""Run one GEMM shape a few times (ncu target).  argv: M N K rate"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_08040_b200 import fbq
M, N, K = (int(a) for a in sys.argv[1:4])
rate = float(sys.argv[4]) if len(sys.argv) > 4 else 0.0
torch.manual_seed(0)
x = torch.randn(M, K, device="cuda"); x[:, 7] *= 100
w = torch.randn(N, K, device="cuda") * 0.02
wq = fbq.transpose(fbq.quantize_rtn(w))
fa = fbq.fallback_quantize(x, fbq.mask_topk(fbq.score_blocks(x), rate))
out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    fbq.fallback_gemm(fa, wq, out=out, exact=False)
torch.cuda.synchronize()

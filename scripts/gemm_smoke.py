"""One small GEMM of each layout, checked against the C oracle; for hang triage."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_08040_b200 import fbq
torch.manual_seed(0)
M, N, K = 256, 256, 384
x = torch.randn(M, K, device="cuda"); w = torch.randn(N, K, device="cuda")
qa = fbq.quantize_rtn(x); wq = fbq.transpose(fbq.quantize_rtn(w))
out = torch.empty(M, N, device="cuda")
fbq.block_quant_gemm(qa, wq, out=out, exact=True); torch.cuda.synchronize()
ref = (fbq.dequantize(qa) @ fbq.dequantize(fbq.quantize_rtn(w)).t())
print("gemm ok, max rel err vs dequant matmul", ((out - ref).abs().max() / ref.abs().max()).item(), flush=True)

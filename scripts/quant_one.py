"""Run the C2 quantizer (8192x14336 bf16, fallback detect at ~5 %) once per K1 variant (ncu target)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_08040_b200 import fbq
import bench
lib = fbq.K.lib
lib.fbq_debug_set_quant_diag.argtypes = [fbq.K.cint]
x = bench.make_activations(8192, 14336, 5, "cuda", torch.bfloat16)
sc = fbq.score_blocks(x).flatten().sort(descending=True).values
theta = float(sc[int(0.05 * sc.numel())].item())
for d in [0, 1]:
    lib.fbq_debug_set_quant_diag(d)
    for _ in range(2):
        fbq.fallback_quantize(x, theta=theta)
torch.cuda.synchronize()

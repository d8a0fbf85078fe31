"""One C2 quantizer launch (ncu target): python scripts/quant_prof.py ROWS COLS bf16|f32 RATE [diag]."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_08040_b200 import fbq
import bench
rows, cols, dt, rate = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], float(sys.argv[4])
diag = int(sys.argv[5]) if len(sys.argv) > 5 else 0
lib = fbq.K.lib
lib.fbq_debug_set_quant_diag.argtypes = [fbq.K.cint]
lib.fbq_debug_set_quant_diag(diag)
x = bench.make_activations(rows, cols, 5, "cuda", torch.bfloat16 if dt == "bf16" else torch.float32)
sc = fbq.score_blocks(x)
mask = fbq.mask_topk(sc, rate) if rate > 0 else torch.zeros_like(sc, dtype=torch.bool)
for _ in range(3):
    fbq.fallback_quantize(x, mask)
torch.cuda.synchronize()

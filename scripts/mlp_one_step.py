"""One warm C3 MLP step (ncu target): bf16, FMA epilogue, T=8192, 4096 -> 14336."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2503_08040_b200 import linear
T, D, Fd = 8192, 4096, 14336
torch.manual_seed(0)
wg = (torch.randn(Fd, D) * 0.02).numpy(); wu = (torch.randn(Fd, D) * 0.02).numpy(); wd = (torch.randn(D, Fd) * 0.02).numpy()
m = linear.GluMlp(wg, wu, wd, T, act_dtype=torch.bfloat16, mid_dtype=torch.bfloat16, exact=False)
x = bench.make_activations(T, D, 3, "cuda", torch.bfloat16)
m.set_thresholds(*bench.mlp_thresholds(x, wg, wu, "cuda"))  # controllers inside their band, as the bench
gy = (torch.randn(T, D, device="cuda") * 1e-3).to(torch.bfloat16)
for step in range(3):
    m.forward(x, step)
    m.backward(gy, step)
torch.cuda.synchronize()

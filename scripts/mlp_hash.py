"""One bench-config MLP step; prints a hash of y, dX and the three dW (cross-build bit-identity checks)."""
import sys, os, hashlib
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2503_08040_b200 import fbq, linear
T = 8192
wg, wu, wd = bench.make_weights()
mlp = linear.GluMlp(wg, wu, wd, T, act_dtype=torch.bfloat16, mid_dtype=torch.bfloat16, exact=False)
x = bench.make_activations(T, bench.D_MODEL, 1000, "cuda", torch.bfloat16)
gy = bench.make_grads(T, bench.D_MODEL, 2000, "cuda", torch.bfloat16)
mlp.set_thresholds(20.0, 2.0)
h = hashlib.sha256()
for i in range(2):
    mlp.zero_grad()
    y = mlp.forward(x, i)
    gx = mlp.backward(gy, i)
    mlp.controller_step()
torch.cuda.synchronize()
for t in [y, gx] + list(mlp.grad_tensors()):
    h.update(t.contiguous().view(torch.uint8).cpu().numpy().tobytes())
print("hash", h.hexdigest()[:16])

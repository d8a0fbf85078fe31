import sys, os
sys.path.insert(0, "/root/repo")
import torch
from paper_2503_08040_b200 import fbq, linear
import bench
T = 8192
wg, wu, wd = bench.make_weights()
mlp = linear.GluMlp(wg, wu, wd, T)
x = bench.make_activations(T, 4096, 1000, "cuda", torch.bfloat16)
gy = bench.make_grads(T, 4096, 2000, "cuda", torch.bfloat16)
mlp.set_thresholds(30.0, 3.0)
for d in [0, 512, 0, 512]:
    fbq.K.lib.fbq_debug_set_quant_diag(d)
    for i in range(3):
        mlp.zero_grad(); mlp.forward(x, i); mlp.backward(gy, i); mlp.controller_step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(10):
        mlp.zero_grad(); mlp.forward(x, i); mlp.backward(gy, i); mlp.controller_step()
    e1.record(); torch.cuda.synchronize()
    print("diag", d, "step ms", e0.elapsed_time(e1) / 10, flush=True)

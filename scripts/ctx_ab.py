"""A/B: C3 step with packed 10-bit vs int16 GluCombine contexts, interleaved repeats."""
import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2503_08040_b200 import linear
T = 8192
wg, wu, wd = bench.make_weights()
x = bench.make_activations(T, 4096, 1000, "cuda", torch.bfloat16)
gy = bench.make_grads(T, 4096, 2000, "cuda", torch.bfloat16)
th = bench.mlp_thresholds(x, wg, wu, "cuda")
ms = {}
for packed in (False, True):
    m = linear.GluMlp(wg, wu, wd, T, act_dtype=torch.bfloat16, mid_dtype=torch.bfloat16, exact=False, ctx_packed=packed)
    m.set_thresholds(*th)
    ms[packed] = m
y, gx = torch.empty_like(x), torch.empty_like(x)
for rep in range(4):
    for packed in (False, True):
        m = ms[packed]; i = [0]
        def step():
            m.zero_grad(); m.forward(x, i[0], out=y); m.backward(gy, i[0], out=gx); m.controller_step(); i[0] += 1
        t = bench._event_time(step, 20, 3)
        print(rep, "packed" if packed else "int16 ", round(T / (t * 1e-3) / 1e6, 4), "M tokens/s", flush=True)

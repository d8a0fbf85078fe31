"""C3 step (zero_grad + fwd + bwd + controller) eager vs replayed from a CUDA graph."""
import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2503_08040_b200 import linear
T = 8192
wg, wu, wd = bench.make_weights()
x = bench.make_activations(T, 4096, 1000, "cuda", torch.bfloat16)
gy = bench.make_grads(T, 4096, 2000, "cuda", torch.bfloat16)
m = linear.GluMlp(wg, wu, wd, T, act_dtype=torch.bfloat16, mid_dtype=torch.bfloat16, exact=False)
m.set_thresholds(*bench.mlp_thresholds(x, wg, wu, "cuda"))
y, gx = torch.empty_like(x), torch.empty_like(x)
def step(i):
    m.zero_grad(); m.forward(x, i, out=y); m.backward(gy, i, out=gx); m.controller_step()
for i in range(3): step(i)
torch.cuda.synchronize()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    step(3)  # warm on the capture stream
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        step(4)
torch.cuda.synchronize()
for rep in range(3):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for i in range(20): step(10 + i)
    e1.record(); torch.cuda.synchronize()
    te = e0.elapsed_time(e1) / 20
    e0.record()
    for i in range(20): g.replay()
    e1.record(); torch.cuda.synchronize()
    tg = e0.elapsed_time(e1) / 20
    print(f"eager {te:.3f} ms ({T / te * 1e-3:.4f} M tok/s)   graph {tg:.3f} ms ({T / tg * 1e-3:.4f} M tok/s)", flush=True)

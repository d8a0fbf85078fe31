"""Does host<->device traffic slow the device step?  The C3 MLP step timed on
the device alone, and again while two other streams keep PCIe busy both ways
with the e2e step's volume (2 x 134 MB each direction per step)."""
import sys, os, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2503_08040_b200 import linear

T = 8192
wg, wu, wd = bench.make_weights()
m = linear.GluMlp(wg, wu, wd, T)
x = bench.make_activations(T, 4096, 1000, "cuda", torch.bfloat16)
gy = bench.make_grads(T, 4096, 2000, "cuda", torch.bfloat16)
m.set_thresholds(*bench.mlp_thresholds(x, wg, wu, "cuda", pooled=False))
y, gx = torch.empty_like(x), torch.empty_like(x)
n = T * 4096
hin = [torch.empty(n, pin_memory=True) for _ in range(2)]
hout = [torch.empty(n, pin_memory=True) for _ in range(2)]
din = [torch.empty(n, device="cuda") for _ in range(2)]
dout = [torch.empty(n, device="cuda") for _ in range(2)]
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
i = [0]


def step():
    m.zero_grad(); m.forward(x, i[0], out=y); m.backward(gy, i[0], out=gx); m.controller_step(); i[0] += 1


def copies():
    with torch.cuda.stream(sa):
        for k in range(2):
            din[k].copy_(hin[k], non_blocking=True)
    with torch.cuda.stream(sb):
        for k in range(2):
            hout[k].copy_(dout[k], non_blocking=True)


for rep in range(3):
    for busy in (False, True):
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(20):
            if busy:
                copies()
            step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        print(f"{'with PCIe traffic' if busy else 'device only      '}: {ms:.3f} ms/step  {T / ms / 1e3:.4f}M tok/s",
              flush=True)

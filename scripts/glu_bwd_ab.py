"""GLU backward: default (two evaluations) vs register-cached 512-thread variant (quant diag 65536):
bit-identical outputs, and C3 step time interleaved."""
import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2503_08040_b200 import linear, fbq
lib = fbq.K.lib; lib.fbq_debug_set_quant_diag.argtypes = [fbq.K.cint]
T = 8192
wg, wu, wd = bench.make_weights()
x = bench.make_activations(T, 4096, 1000, "cuda", torch.bfloat16)
gy = bench.make_grads(T, 4096, 2000, "cuda", torch.bfloat16)
th = bench.mlp_thresholds(x, wg, wu, "cuda")
outs = {}
for d in (0, 65536):
    lib.fbq_debug_set_quant_diag(d)
    m = linear.GluMlp(wg, wu, wd, T, act_dtype=torch.bfloat16, mid_dtype=torch.bfloat16, exact=False)
    m.set_thresholds(*th)
    y = m.forward(x, 0); g = m.backward(gy, 0); torch.cuda.synchronize()
    outs[d] = (y.clone(), g.clone(), [t.clone() for t in m.grad_tensors()])
    del m
lib.fbq_debug_set_quant_diag(0)
same = torch.equal(outs[0][0], outs[65536][0]) and torch.equal(outs[0][1], outs[65536][1]) and \
    all(torch.equal(a.view(torch.int32), b.view(torch.int32)) for a, b in zip(outs[0][2], outs[65536][2]))
print("bit-identical:", same, flush=True)
m = linear.GluMlp(wg, wu, wd, T, act_dtype=torch.bfloat16, mid_dtype=torch.bfloat16, exact=False)
m.set_thresholds(*th)
y, gx = torch.empty_like(x), torch.empty_like(x)
for rep in range(3):
    for d in (0, 65536):
        lib.fbq_debug_set_quant_diag(d)
        i = [0]
        def step():
            m.zero_grad(); m.forward(x, i[0], out=y); m.backward(gy, i[0], out=gx); m.controller_step(); i[0] += 1
        t = bench._event_time(step, 20, 3)
        print(rep, d, round(T / (t * 1e-3) / 1e6, 4), "M tok/s", flush=True)
lib.fbq_debug_set_quant_diag(0)

"""Same-process A/B of kernel variants inside the C3 MLP step (K1 diag flags, or GEMM diag flags with AB_GEMM=1)
(Llama-3.1-8B SwiGLU, 8192 tokens, bf16, bench thresholds): K1 diag flags from
the command line, interleaved; outputs must be bit-identical across flags."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2503_08040_b200 import fbq, linear
lib = fbq.K.lib
lib.fbq_debug_set_quant_diag.argtypes = [fbq.K.cint]
lib.fbq_debug_set_gemm_diag.argtypes = [fbq.K.cint]
SET = lib.fbq_debug_set_gemm_diag if os.environ.get("AB_GEMM") else lib.fbq_debug_set_quant_diag
diags = [int(a) for a in sys.argv[1:]] or [0, 32]
T = 8192
wg, wu, wd = bench.make_weights()
mlp = linear.GluMlp(wg, wu, wd, T, act_dtype=torch.bfloat16, mid_dtype=torch.bfloat16, exact=False)
x = bench.make_activations(T, bench.D_MODEL, 1000, "cuda", torch.bfloat16)
gy = bench.make_grads(T, bench.D_MODEL, 2000, "cuda", torch.bfloat16)
th_gu = float(torch.quantile(fbq.score_blocks(x).flatten(), 0.85))
with torch.no_grad():
    xs = x[:1024].float()
    h = torch.nn.functional.silu(xs @ torch.from_numpy(wg).cuda().t()) * (xs @ torch.from_numpy(wu).cuda().t())
    th_d = float(torch.quantile(fbq.score_blocks(h).flatten(), 0.85))
    del xs, h
y = torch.empty_like(x)
gx = torch.empty_like(x)


def step(i):
    mlp.zero_grad()
    mlp.forward(x, i, 0, out=y)
    mlp.backward(gy, i, 0, out=gx)


res, outs = {d: [] for d in diags}, {}
for rnd in range(3):
    for d in diags:
        SET(d)
        mlp.set_thresholds(th_gu, th_d)
        for i in range(2):
            step(i)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(10):
            step(i)
        e1.record()
        torch.cuda.synchronize()
        res[d].append(e0.elapsed_time(e1) / 10)
        mlp.set_thresholds(th_gu, th_d)
        step(0)
        torch.cuda.synchronize()
        outs[d] = (y.clone(), gx.clone(), [g.clone() for g in mlp.grad_tensors()])
SET(0)
for d in diags:
    print(f"diag={d:3d}: ms/step {' '.join(f'{v:.3f}' for v in res[d])}  best {T/min(res[d])*1e3/1e6:.4f}M tokens/s")
ref = outs[diags[0]]
for d in diags[1:]:
    o = outs[d]
    same = torch.equal(o[0], ref[0]) and torch.equal(o[1], ref[1]) and all(torch.equal(a, b) for a, b in zip(o[2], ref[2]))
    print(f"diag={d} outputs identical to diag={diags[0]}: {same}")

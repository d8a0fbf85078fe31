"""A/B helper for the GEMM output-store path: block GEMMs at the step's shapes
(bf16 and fp32 outputs), the C5 fallback GEMM at 10 % and one MLP step."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2503_08040_b200 import fbq, linear


def timeit(fn, iters=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e-3


out = []
for (M, N, K, dt) in [(8192, 14336, 4096, torch.bfloat16), (4096, 14336, 8192, torch.float32),
                      (8192, 4096, 28672, torch.bfloat16)]:
    x = torch.randn(M, K, device="cuda")
    w = torch.randn(N, K, device="cuda") * 0.02
    qa, wq = fbq.quantize_rtn(x), fbq.transpose(fbq.quantize_rtn(w))
    y = torch.empty(M, N, device="cuda", dtype=dt)
    t = timeit(lambda: fbq.block_quant_gemm(qa, wq, out=y, exact=False))
    out.append(f"{M}x{N}x{K} {str(dt)[6:]} {2 * M * N * K / t / 1e12:.0f}")
M, N, K = 8192, 28672, 8192
x = bench.make_activations(M, K, 11, "cuda", torch.bfloat16)
wq = fbq.transpose(fbq.quantize_rtn(torch.randn(N, K, device="cuda") * 0.02))
fa = fbq.fallback_quantize(x, fbq.mask_topk(fbq.score_blocks(x), 0.10))
y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
t = timeit(lambda: fbq.fallback_gemm(fa, wq, out=y, exact=False), iters=10)
out.append(f"C5@10% {2 * M * N * K / t / 1e12:.0f}")
del x, wq, fa, y
torch.cuda.empty_cache()
T = 8192
wg, wu, wd = bench.make_weights()
m = linear.GluMlp(wg, wu, wd, T)
xa = bench.make_activations(T, 4096, 1000, "cuda", torch.bfloat16)
gy = bench.make_grads(T, 4096, 2000, "cuda", torch.bfloat16)
m.set_thresholds(*bench.mlp_thresholds(xa, wg, wu, "cuda", pooled=False))
ya, gx = torch.empty_like(xa), torch.empty_like(xa)
i = [0]


def step():
    m.zero_grad(); m.forward(xa, i[0], out=ya); m.backward(gy, i[0], out=gx); m.controller_step(); i[0] += 1


t = timeit(step, iters=10)
out.append(f"MLP {T / t / 1e6:.4f}M tok/s")
print("  ".join(out), flush=True)

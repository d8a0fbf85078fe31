"""Tiny driver for ncu captures: one kernel family per invocation."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_08040_b200 import fbq

what = sys.argv[1]
torch.manual_seed(0)
if what == "gemm":
    M, N, K = [int(v) for v in sys.argv[2:5]] if len(sys.argv) > 4 else (8192, 14336, 4096)
    x = torch.randn(M, K, device="cuda"); x[:, 7] *= 100
    w = torch.randn(N, K, device="cuda") * 0.02
    wq = fbq.transpose(fbq.quantize_rtn(w))
    fa = fbq.fallback_quantize(x, fbq.mask_topk(fbq.score_blocks(x), 0.1))
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        fbq.fallback_gemm(fa, wq, out=out, exact=False)
elif what == "rtn32":
    w = torch.randn(4096, 14336, device="cuda") * 0.02
    for _ in range(3):
        fbq.quantize_rtn(w)
elif what == "quant":
    R, C = 8192, 14336
    x = torch.randn(R, C, device="cuda").to(torch.bfloat16)
    for _ in range(3):
        fbq.quantize_rtn(x)
    for _ in range(2):
        fbq.quantize_stochastic(x, 5)
    for _ in range(2):
        fbq.fallback_quantize(x, theta=4.2)
torch.cuda.synchronize()
if what == "mlp":
    import bench
    from paper_2503_08040_b200 import linear
    T = 8192
    wg, wu, wd = bench.make_weights()
    mlp = linear.GluMlp(wg, wu, wd, T, act_dtype=torch.bfloat16, mid_dtype=torch.bfloat16, exact=False)
    x = bench.make_activations(T, bench.D_MODEL, 1000, "cuda", torch.bfloat16)
    gy = bench.make_grads(T, bench.D_MODEL, 2000, "cuda", torch.bfloat16)
    # the bench's calibration: 85th percentile of the block AbsMax of X and of h
    th_gu = float(torch.quantile(fbq.score_blocks(x).flatten(), 0.85))
    with torch.no_grad():
        xs = x[:1024].float()
        h = torch.nn.functional.silu(xs @ torch.from_numpy(wg).cuda().t()) * (xs @ torch.from_numpy(wu).cuda().t())
        th_d = float(torch.quantile(fbq.score_blocks(h).flatten(), 0.85))
        del xs, h
    mlp.set_thresholds(th_gu, th_d)
    for i in range(2):
        mlp.zero_grad(); mlp.forward(x, i); mlp.backward(gy, i); mlp.controller_step()
    torch.cuda.synchronize()

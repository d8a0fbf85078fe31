"""One C5 fallback GEMM launch per mask (topk = bench, random, even rows) for
ncu: which resource makes spread-out fallback blocks expensive?"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_08040_b200 import fbq
import bench

M, N, K = 8192, 28672, 8192
x = bench.make_activations(M, K, 1, "cuda", torch.float32)
w = torch.randn(N, K, device="cuda") * 0.02
wq = fbq.transpose(fbq.quantize_rtn(w))
out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
scores = fbq.score_blocks(x)
MB, KB = scores.shape
g = torch.Generator(device="cpu").manual_seed(0)
n = int(round(0.1 * MB * KB))
r = torch.zeros(MB * KB, dtype=torch.uint8)
r[torch.randperm(MB * KB, generator=g)[:n]] = 1
masks = {"zero": torch.zeros(MB, KB, dtype=torch.uint8, device="cuda"),
         "topk": fbq.mask_topk(scores, 0.1), "random": r.view(MB, KB).cuda()}
for name in os.environ.get("MASKS", "zero,topk,random").split(","):
    fa = fbq.fallback_quantize(x, masks[name])
    for _ in range(2):
        fbq.fallback_gemm(fa, wq, out=out, exact=False)
    torch.cuda.synchronize()
    print(name, flush=True)

"""Clock-independent cost of fallback items on C5: MMA-warp cycles per item and the epilogue timeline
(kProf instance: fbq_debug_set_gemm_prof), 0 % vs 10 % fallback."""
import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2503_08040_b200 import fbq as F
lib = F.K.lib
lib.fbq_debug_set_gemm_prof.argtypes = [F.K.vp]
M, N, K = 8192, 28672, 8192
x = bench.make_activations(M, K, 11, "cuda", torch.bfloat16)
wq = F.transpose(F.quantize_rtn(torch.randn(N, K, device="cuda") * 0.02))
sc = F.score_blocks(x)
y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
prof = torch.zeros(148 * 16, dtype=torch.int64, device="cuda")
for rate in (0.0, 0.1, 0.0, 0.1):
    fa = F.fallback_quantize(x, F.mask_topk(sc, rate))
    for _ in range(3): F.fallback_gemm(fa, wq, out=y, exact=False)
    prof.zero_()
    lib.fbq_debug_set_gemm_prof(prof.data_ptr())
    F.fallback_gemm(fa, wq, out=y, exact=False)
    torch.cuda.synchronize()
    lib.fbq_debug_set_gemm_prof(None)
    pr = prof.view(148, 16).double().cpu()
    items = pr[:, 9]
    mma = pr[:, 0] / items
    tw, tl, tpre, tpost = [(pr[:, 1 + k] / items).mean().item() for k in range(4)]
    print(f"rate {rate:.2f}: items/CTA {items.mean():.0f}  MMA-warp cycles/item {mma.mean():.0f} (min {mma.min():.0f} max {mma.max():.0f})"
          f"  epilogue per item: wait {tw:.0f} ld {tl:.0f} pre-release {tpre:.0f} post {tpost:.0f}", flush=True)

"""One launch per shape for `ncu --metrics dram__bytes_read.sum,...` (raster traffic)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_08040_b200 import fbq
import bench
lib = fbq.K.lib
lib.fbq_debug_set_gemm_diag.argtypes = [fbq.K.cint]
lib.fbq_debug_set_gemm_diag(int(os.environ.get("DIAG", "0"), 0))
for (M, N, K) in [(8192, 28672, 8192), (8192, 4096, 14336), (8192, 4096, 28672), (8192, 28672, 4096)]:
    x = bench.make_activations(M, K, 3, "cuda", torch.bfloat16)
    wq = fbq.transpose(fbq.quantize_rtn(torch.randn(N, K, device="cuda") * 0.02))
    fa = fbq.fallback_quantize(x, fbq.mask_topk(fbq.score_blocks(x), 0.10))
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    fbq.fallback_gemm(fa, wq, out=out, exact=False)
    torch.cuda.synchronize()
    print(M, N, K, "operands MB", round((M * K + N * K) / 2**20), flush=True)
    del x, wq, fa, out
    torch.cuda.empty_cache()

"""The MLP's dX GEMM alone (dG [8192 x 28672] K-major x W_gu [28672 x 4096] MN-major, bf16 out):
TOPS under the chunked-B raster (diag 0) and the old kGroupM groups (diag 1<<27); ncu target."""
import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_08040_b200 import fbq as F
lib = F.K.lib
lib.fbq_debug_set_gemm_diag.argtypes = [F.K.cint]
M, N, K = 8192, 4096, 28672
torch.manual_seed(0)
g = torch.randn(M, K, device="cuda", dtype=torch.bfloat16) * 1e-3
w = torch.randn(K, N, device="cuda") * 0.02
qa = F.quantize_stochastic(g, 77)
qb = F.quantize_rtn(w)
out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
reps = int(os.environ.get("REPS", "10"))
for d in [int(a) for a in sys.argv[1:]] or [0, 1 << 27]:
    lib.fbq_debug_set_gemm_diag(d)
    for _ in range(2):
        F.block_quant_gemm(qa, qb, out=out, exact=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        F.block_quant_gemm(qa, qb, out=out, exact=False)
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps * 1e-3
    print(f"diag {d:#x}: {2*M*N*K/t/1e12:.0f} TOPS ({t*1e3:.3f} ms)", flush=True)
lib.fbq_debug_set_gemm_diag(0)

"""RmsNorm -> linear-input quantizer at the C3/C4 block input (8192 x 4096 bf16, threshold, two SR planes):
fused (y never materialised) vs forward() + fbq_cuda_quantize_linear_input(y)."""
import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2503_08040_b200 import fbq
from paper_2503_08040_b200 import _capi as K
T, D = 8192, 4096
x = bench.make_activations(T, D, 3, "cuda", torch.bfloat16)
n = fbq.RmsNorm(D)
theta = float(fbq.score_blocks(n.forward(x)).flatten().quantile(0.85).item())
nb = (T // 128) * (D // 128)
codes = torch.empty(T, D, dtype=torch.int8, device="cuda"); res = torch.empty_like(codes)
sr1, sr2 = torch.empty_like(codes), torch.empty_like(codes)
sc = torch.empty(nb, device="cuda"); rsc = torch.empty_like(sc)
bits = torch.empty((nb + 31) // 32, dtype=torch.int32, device="cuda"); cnt = torch.empty(1, dtype=torch.int32, device="cuda")
ctx = torch.empty(T, D, dtype=torch.int16, device="cuda"); ctx_s = torch.empty(T, D // 128, device="cuda")
rms = torch.empty(T, device="cuda"); st = torch.cuda.current_stream().cuda_stream
def unfused():
    y = n.forward(x)
    K.call("fbq_cuda_quantize_linear_input", y.data_ptr(), K.FBQ_BF16, T, D, D, K.FBQ_MASK_THRESHOLD, theta, None,
           bits.data_ptr(), codes.data_ptr(), D, sc.data_ptr(), res.data_ptr(), rsc.data_ptr(), cnt.data_ptr(),
           sr1.data_ptr(), 11, sr2.data_ptr(), 12, 0, st)
def fused():
    K.call("fbq_cuda_rmsnorm_quantize_input", x.data_ptr(), K.FBQ_BF16, T, D, D, n.gain.data_ptr(), ctx.data_ptr(), D,
           ctx_s.data_ptr(), rms.data_ptr(), K.FBQ_MASK_THRESHOLD, theta, None, bits.data_ptr(), codes.data_ptr(), D,
           sc.data_ptr(), res.data_ptr(), rsc.data_ptr(), cnt.data_ptr(), sr1.data_ptr(), 11, sr2.data_ptr(), 12, 0, st)
for rep in range(2):
    for name, fn in (("unfused", unfused), ("fused", fused)):
        t = bench._event_time(fn, 20, 3)
        print(rep, name, round(t * 1e3, 1), "us", flush=True)

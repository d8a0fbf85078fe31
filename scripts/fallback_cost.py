"""Where the fallback items' extra cost goes on C5: TOPS at 0 / 10 % with the full epilogue and with the
epilogue math skipped (diag 1), plus the median SM clock (NVML) over each timed loop."""
import sys, os, threading, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2503_08040_b200 import fbq as F
import pynvml
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
lib = F.K.lib; lib.fbq_debug_set_gemm_diag.argtypes = [F.K.cint]
M, N, K = 8192, 28672, 8192
x = bench.make_activations(M, K, 11, "cuda", torch.bfloat16)
wq = F.transpose(F.quantize_rtn(torch.randn(N, K, device="cuda") * 0.02))
sc = F.score_blocks(x)
y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
def run(fa, reps=20):
    for _ in range(3): F.fallback_gemm(fa, wq, out=y, exact=False)
    torch.cuda.synchronize()
    clk = []; stop = [False]
    def samp():
        while not stop[0]:
            clk.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)); time.sleep(0.005)
    th = threading.Thread(target=samp); th.start()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps): F.fallback_gemm(fa, wq, out=y, exact=False)
    e1.record(); torch.cuda.synchronize(); stop[0] = True; th.join()
    t = e0.elapsed_time(e1) / reps * 1e-3
    clk.sort()
    return 2 * M * N * K / t / 1e12, clk[len(clk) // 2] if clk else None
for rate in (0.0, 0.1):
    fa = F.fallback_quantize(x, F.mask_topk(sc, rate))
    for d, name in ((0, "epilogue"), (1, "no-epi-math"), (3, "no-epi-math, no TMA"), (2, "no TMA")):
        lib.fbq_debug_set_gemm_diag(d)
        tops, mhz = run(fa)
        print(f"rate {rate:.2f} {name:22s}: {tops:7.1f} TOPS  median SM {mhz} MHz", flush=True)
lib.fbq_debug_set_gemm_diag(0)

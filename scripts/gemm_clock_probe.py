"""Per-item MMA-warp cycles vs wall time and SM clocks under sustained load:
is the GEMM latency-bound (cycles/item >> 512) or clock/power-bound?"""
import sys, os, subprocess, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_08040_b200 import fbq

lib = fbq.K.lib
lib.fbq_debug_set_gemm_prof.argtypes = [fbq.K.vp]


def sample_clocks(stop, out):
    while not stop.is_set():
        r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active",
                            "--format=csv,noheader,nounits", "-i", "0"], capture_output=True, text=True)
        out.append(r.stdout.strip())
        time.sleep(0.05)


def loaded(fn, seconds=1.5):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); fn(); e.record(); torch.cuda.synchronize()
    one = s.elapsed_time(e) * 1e-3
    n = max(3, int(seconds / one))
    stop, clk = threading.Event(), []
    th = threading.Thread(target=sample_clocks, args=(stop, clk)); th.start()
    s.record()
    for _ in range(n):
        fn()
    e.record(); torch.cuda.synchronize()
    stop.set(); th.join()
    return s.elapsed_time(e) * 1e-3 / n, clk[len(clk) // 4: 3 * len(clk) // 4 + 1]


M, N, K = 8192, 14336, 4096
torch.manual_seed(0)
x = torch.randn(M, K, device="cuda")
w = torch.randn(N, K, device="cuda") * 0.02
wq = fbq.transpose(fbq.quantize_rtn(w))
qa = fbq.quantize_rtn(x)
out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
ops = 2 * M * N * K
t, clk = loaded(lambda: fbq.block_quant_gemm(qa, wq, out=out, exact=False))
print(f"fbq gemm: {t*1e3:.3f} ms {ops/t/1e12:.0f} TOPS clocks {clk[:6]}", flush=True)
prof = torch.zeros(148 * 16, dtype=torch.int64, device="cuda")
for exact in (False, True):
    prof.zero_()
    lib.fbq_debug_set_gemm_prof(prof.data_ptr())
    fbq.block_quant_gemm(qa, wq, out=out, exact=exact)
    torch.cuda.synchronize()
    lib.fbq_debug_set_gemm_prof(None)
    pr = prof.view(148, 16).double()
    items = pr[:, 9].mean().item()
    print(f"exact={exact} MMA warp cycles/CTA {pr[:,0].mean().item():.0f} items/CTA {items:.0f} -> per item {pr[:,0].mean().item()/items:.0f}", flush=True)
    for h in (0, 1):
        w, l, pre, post = [(pr[:, 1 + 4 * h + k].mean().item() / items) for k in range(4)]
        print(f"  epilogue h={h} per item: wait-tfull {w:.0f}  tmem-ld(2 chunks) {l:.0f}  to-release {pre:.0f}  after-release {post:.0f}  total {w+l+pre+post:.0f}", flush=True)
xi = torch.randint(-127, 127, (M, K), device="cuda", dtype=torch.int8)
wi = torch.randint(-127, 127, (K, N), device="cuda", dtype=torch.int8)
t, clk = loaded(lambda: torch._int_mm(xi, wi))
print(f"cuBLAS int8: {t*1e3:.3f} ms {ops/t/1e12:.0f} TOPS clocks {clk[:6]}", flush=True)
xb = x.to(torch.bfloat16); wb = w.to(torch.bfloat16)
t, clk = loaded(lambda: xb @ wb.t())
print(f"cuBLAS bf16: {t*1e3:.3f} ms {ops/t/1e12:.0f} TFLOPS clocks {clk[:6]}", flush=True)

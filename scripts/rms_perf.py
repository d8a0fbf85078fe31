"""RMSNorm fwd/bwd timing at the Llama-3.1-8B shape (8192 x 4096), CUDA events; per-kernel via the profiler-free event split."""
import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_08040_b200 import fbq as F
import bench

def timeit(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3  # us

for dt in (torch.bfloat16, torch.float32):
    x = bench.make_activations(8192, 4096, 3, "cuda", dt)
    n = F.RmsNorm(4096)
    gy = (torch.randn(8192, 4096, device="cuda") * 1e-3).to(dt)
    tf = timeit(lambda: n.forward(x))
    tb = timeit(lambda: n.backward(gy))
    tq = timeit(lambda: F.fallback_quantize(x, theta=4.0))
    print(f"{dt}: rmsnorm fwd {tf:.1f} us, bwd {tb:.1f} us; K1 on x (for scale) {tq:.1f} us", flush=True)

"""The bench's e2e leg alone (host fp32 buffers through fbq_mlp_step_host_async), repeated."""
import sys, os, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2503_08040_b200 import linear
T = 8192
wg, wu, wd = bench.make_weights()
x = bench.make_activations(T, 4096, 1000, "cuda", torch.bfloat16)
gy = bench.make_grads(T, 4096, 2000, "cuda", torch.bfloat16)
th = bench.mlp_thresholds(x, wg, wu, "cuda")
xh = x.float().cpu().pin_memory(); gyh = gy.float().cpu().pin_memory()
yh = torch.empty_like(xh).pin_memory(); gxh = torch.empty_like(xh).pin_memory()
m = linear.GluMlp(wg, wu, wd, T, act_dtype=torch.float32, mid_dtype=torch.bfloat16, exact=False)
m.set_thresholds(*th)
flags = m.STEP_ZERO_GRAD | m.STEP_CONTROLLER
for i in range(2): m.step_host_async(xh, gyh, i, yh, gxh, flags)
m.host_sync()
for rep in range(3):
    t0 = time.perf_counter()
    for i in range(30): m.step_host_async(xh, gyh, 2 + i, yh, gxh, flags)
    m.host_sync()
    dt = (time.perf_counter() - t0) / 30
    print("e2e", round(T / dt / 1e6, 4), "M tok/s", flush=True)
# H2D / D2H bandwidth of this box
a = torch.empty(T * 4096, device="cuda")
for name, fn in (("h2d", lambda: a.copy_(xh.view(-1), non_blocking=True)), ("d2h", lambda: yh.view(-1).copy_(a, non_blocking=True))):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(10): fn()
    torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 10
    print(name, round(T * 4096 * 4 / dt / 1e9, 1), "GB/s", flush=True)

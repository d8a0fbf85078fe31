"""PCIe bandwidth of this box: H2D alone, D2H alone, and both at once (the e2e
step's pattern: 2 x 134 MB fp32 in and 2 x 134 MB out per step), pinned buffers."""
import time, torch
n = 8192 * 4096
hin = [torch.empty(n, pin_memory=True) for _ in range(2)]
hout = [torch.empty(n, pin_memory=True) for _ in range(2)]
din = [torch.empty(n, device="cuda") for _ in range(2)]
dout = [torch.empty(n, device="cuda") for _ in range(2)]
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()


def run(h2d, d2h, reps=10):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        if h2d:
            with torch.cuda.stream(sa):
                for i in range(2):
                    din[i].copy_(hin[i], non_blocking=True)
        if d2h:
            with torch.cuda.stream(sb):
                for i in range(2):
                    hout[i].copy_(dout[i], non_blocking=True)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


for _ in range(2):
    run(True, True, 2)
b = 2 * n * 4
for name, h, d in (("h2d alone", True, False), ("d2h alone", False, True), ("both at once", True, True)):
    t = run(h, d)
    print(f"{name:13s} {t * 1e3:6.2f} ms per step-pattern ({b / 1e6:.0f} MB each way)  "
          f"{b / t / 1e9:5.1f} GB/s per direction", flush=True)

"""apply_sgd fused with the weight RTN (one pass) vs the update then the RTN
(two passes), on the C3 weight shapes (fp32 master weights), CUDA events."""
import sys, os, json, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2503_08040_b200 import _capi as K
peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
s = torch.cuda.current_stream()
for (R, C) in [(28672, 4096), (4096, 14336)]:
    w = torch.randn(R, C, device="cuda") * 0.02
    g = torch.randn(R, C, device="cuda")
    q = torch.empty(R, C, dtype=torch.int8, device="cuda")
    sc = torch.empty((R // 128) * (C // 128), device="cuda")
    fused = lambda: K.call("fbq_cuda_sgd_quantize_rtn", w.data_ptr(), g.data_ptr(), R, C, 1e-6, q.data_ptr(), C,
                           sc.data_ptr(), s.cuda_stream)

    def two():
        K.call("fbq_cuda_sgd_update", w.data_ptr(), g.data_ptr(), R * C, 1e-6, s.cuda_stream)
        K.call("fbq_cuda_quantize_rtn", w.data_ptr(), K.FBQ_F32, R, C, C, q.data_ptr(), C, sc.data_ptr(),
               s.cuda_stream)
    rtn = lambda: K.call("fbq_cuda_quantize_rtn", w.data_ptr(), K.FBQ_F32, R, C, C, q.data_ptr(), C,
                         sc.data_ptr(), s.cuda_stream)
    n = R * C
    for name, fn, byt in [("fused sgd+rtn", fused, n * 13), ("sgd then rtn", two, n * 17), ("rtn alone", rtn, n * 5)]:
        t = bench._events_time(fn, s, n=10)
        print(f"{R}x{C} {name:14s} {t * 1e6:8.1f} us  {byt / t / 1e9:7.0f} GB/s  {byt / t / 1e9 / peak:.3f} of HBM", flush=True)

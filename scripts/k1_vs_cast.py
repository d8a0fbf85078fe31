"""K1 (quantize + fallback detect at 0 %) next to the plainest streaming kernel
with the same traffic: torch's elementwise cast x -> int8 into a preallocated
buffer (reads x once, writes one byte per element).  Both timed back to back
with CUDA events like bench.quant_sweep; rows swept to fit t = t0 + bytes / BW."""
import sys, os, json, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2503_08040_b200 import fbq
from paper_2503_08040_b200 import _capi as K

stream = torch.cuda.current_stream()
peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]


def timeit(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(stream)
    for _ in range(n):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e-3


out = {}
for dt in (torch.bfloat16, torch.float32):
    for (R, C) in [(2048, 4096), (4096, 4096), (8192, 4096), (16384, 4096), (8192, 14336), (32768, 4096)]:
        nb = (R // 128) * (C // 128)
        x = bench.make_activations(R, C, 5, "cuda", dt)
        codes = torch.empty(R, C, dtype=torch.int8, device="cuda")
        res = torch.empty_like(codes)
        scales = torch.empty(nb, device="cuda")
        rscales = torch.empty_like(scales)
        bits = torch.zeros((nb + 31) // 32, dtype=torch.int32, device="cuda")
        count = torch.zeros(1, dtype=torch.int32, device="cuda")
        theta = float(fbq.score_blocks(x).max().item()) * 2.0  # 0 % fallback

        def k1():
            K.call("fbq_cuda_quantize_fallback", x.data_ptr(), K.FBQ_BF16 if dt == torch.bfloat16 else K.FBQ_F32,
                   R, C, C, K.FBQ_MASK_THRESHOLD, theta, bits.data_ptr(), codes.data_ptr(), C,
                   scales.data_ptr(), res.data_ptr(), rscales.data_ptr(), count.data_ptr(),
                   None, None, 0, 0, stream.cuda_stream)

        def cast():
            codes.copy_(x)

        byt = R * C * (x.element_size() + 1)
        tk, tc = timeit(k1), timeit(cast)
        key = f"{R}x{C} {str(dt)[6:]}"
        out[key] = {"MB": round(byt / 1e6, 1), "k1_us": round(tk * 1e6, 2), "cast_us": round(tc * 1e6, 2),
                    "k1_frac": round(byt / tk / 1e9 / peak, 3), "cast_frac": round(byt / tc / 1e9 / peak, 3)}
        print(key, out[key], flush=True)
        del x, codes, res
print(json.dumps(out))

"""C2 quantizer sweep: quantize + fallback-detect on Llama-3.1-8B activation
shapes at fallback ratios 0/5/20 % (bf16 and fp32), GB/s of algorithmic bytes
(in + codes + residual codes of flagged blocks + scales + bitmap), plus the
RTN weight quantizer and the stochastic (context) quantizer; persistent TMA K1
vs the one-block-per-CTA K1 (diag 1)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_08040_b200 import fbq
import bench

lib = fbq.K.lib
lib.fbq_debug_set_quant_diag.argtypes = [fbq.K.cint]


def timeit(fn, iters=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e-3


peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
res = {}
DIAGS = [int(a) for a in sys.argv[1:]] or [0, 1]
for (R, C) in [(8192, 4096), (8192, 14336)]:
    for dt in [torch.bfloat16, torch.float32]:
        x = bench.make_activations(R, C, 5, "cuda", dt)
        esz = x.element_size()
        nb = (R // 128) * (C // 128)
        sc = fbq.score_blocks(x).flatten().sort(descending=True).values
        for rate in [0.0, 0.05, 0.20]:
            k = int(round(rate * nb))
            theta = float(sc[k].item()) if k < nb else 0.0  # exactly k blocks strictly above
            if rate == 0.0:
                theta = float(sc[0].item())
            for diag in DIAGS:
                lib.fbq_debug_set_quant_diag(diag)
                t = timeit(lambda: fbq.fallback_quantize(x, theta=theta))
                fa = fbq.fallback_quantize(x, theta=theta)
                f = int(fa.masked_count.item()) / nb if fa.masked_count is not None else rate
                byt = R * C * (esz + 1) + f * R * C + nb * 4 * (1 + f) + nb / 8
                res[f"fallback {R}x{C} {str(dt)[6:]} rate={rate:.2f} d{diag}"] = \
                    f"{t*1e6:7.1f} us {byt/t/1e9:6.0f} GB/s ({byt/t/1e9/peak*100:4.1f}% HBM)"
        for diag in DIAGS:
            lib.fbq_debug_set_quant_diag(diag)
            t = timeit(lambda: fbq.quantize_rtn(x))
            byt = R * C * (esz + 1) + nb * 4
            res[f"rtn {R}x{C} {str(dt)[6:]} d{diag}"] = f"{t*1e6:7.1f} us {byt/t/1e9:6.0f} GB/s ({byt/t/1e9/peak*100:4.1f}% HBM)"
            t = timeit(lambda: fbq.quantize_stochastic(x, 1234))
            res[f"sr {R}x{C} {str(dt)[6:]} d{diag}"] = f"{t*1e6:7.1f} us {byt/t/1e9:6.0f} GB/s ({byt/t/1e9/peak*100:4.1f}% HBM)"
        lib.fbq_debug_set_quant_diag(0)
        del x
for k, v in res.items():
    print(f"{k:48s} {v}")
json.dump(res, open("gpurun_out/quant_perf.json", "w"), indent=1)

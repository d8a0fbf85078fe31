"""A/B: stochastic-context quantizer launches on the smem-staged K1
(default) vs the register-resident K1 (diag 8): dY SR (1 plane) and the linear
input (RTN + fallback detect + 2 SR planes), Llama-8B MLP shapes, bf16."""
import sys, os
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


for (R, C) in [(8192, 4096), (8192, 14336)]:
    for dt in (torch.bfloat16, torch.float32):
        x = bench.make_activations(R, C, 5, "cuda", dt)
        sc = fbq.score_blocks(x).flatten().sort(descending=True).values
        theta = float(sc[int(0.05 * sc.numel())].item())
        res = {}
        for d in (0, 8):
            lib.fbq_debug_set_quant_diag(d)
            q1 = fbq.quantize_stochastic(x, 1234, row_offset=256)
            f2, c2 = fbq.fallback_quantize(x, theta=theta, sr_seed=99)
            res[d] = (q1.codes.clone(), f2.primary.codes.clone(), c2.codes.clone(), f2.mask_bits.clone())
            t1 = timeit(lambda: fbq.quantize_stochastic(x, 1234))
            t2 = timeit(lambda: fbq.fallback_quantize(x, theta=theta, sr_seed=99))
            byt1 = R * C * (x.element_size() + 1)
            print(f"{R}x{C} {str(dt)[6:]} diag={d}: SR {t1*1e6:7.1f} us ({byt1/t1/1e9:5.0f} GB/s)  "
                  f"fallback+SR {t2*1e6:7.1f} us", flush=True)
        lib.fbq_debug_set_quant_diag(0)
        assert all(torch.equal(a, b) for a, b in zip(res[0], res[8])), "reg vs smem K1 differ"

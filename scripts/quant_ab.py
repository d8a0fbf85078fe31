"""Same-process A/B of K1 variants on the C2 bf16 cases (fallback detect at
5 %): diag flags given on the command line, interleaved over 3 rounds."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_08040_b200 import fbq
from paper_2503_08040_b200 import _capi as K
import bench
lib = fbq.K.lib
lib.fbq_debug_set_quant_diag.argtypes = [fbq.K.cint]
diags = [int(a) for a in sys.argv[1:]] or [0, 16]
stream = torch.cuda.current_stream()
for (R, C) in [(8192, 4096), (8192, 14336)]:
    x = bench.make_activations(R, C, 5, "cuda", torch.bfloat16)
    nb = (R // 128) * (C // 128)
    sc = fbq.score_blocks(x).flatten().sort(descending=True).values
    theta = float(sc[int(0.05 * nb)].item())
    codes = torch.empty(R, C, dtype=torch.int8, device="cuda")
    res = torch.empty_like(codes)
    scales = torch.empty(nb, dtype=torch.float32, device="cuda")
    rscales = torch.empty_like(scales)
    bits = torch.zeros((nb + 31) // 32, dtype=torch.int32, device="cuda")
    count = torch.zeros(1, dtype=torch.int32, device="cuda")

    def run():
        K.call("fbq_cuda_quantize_fallback", x.data_ptr(), K.FBQ_BF16, R, C, C, K.FBQ_MASK_THRESHOLD, theta,
               bits.data_ptr(), codes.data_ptr(), C, scales.data_ptr(), res.data_ptr(), rscales.data_ptr(),
               count.data_ptr(), None, None, 0, 0, stream.cuda_stream)
    out = {d: [] for d in diags}
    for rnd in range(3):
        for d in diags:
            lib.fbq_debug_set_quant_diag(d)
            for _ in range(3):
                run()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(30):
                run()
            e1.record(stream)
            torch.cuda.synchronize()
            out[d].append(e0.elapsed_time(e1) / 30 * 1e3)
    lib.fbq_debug_set_quant_diag(0)
    byt = R * C * 3 + 0.05 * R * C
    for d, ts in out.items():
        t = min(ts)
        print(f"{R}x{C} bf16 diag={d:3d}: {' '.join(f'{v:6.1f}' for v in ts)} us  best {byt/t/1e3:6.0f} GB/s", flush=True)

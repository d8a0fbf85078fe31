"""Fixed per-call overhead of K1 on small shapes: with vs without the masked-count zeroing grid (PDL)."""
import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2503_08040_b200 import fbq
from paper_2503_08040_b200 import _capi as K
stream = torch.cuda.current_stream()
for (R, C) in [(8192, 4096), (8192, 14336)]:
    nb = (R // 128) * (C // 128)
    codes = torch.empty(R, C, dtype=torch.int8, device="cuda"); res = torch.empty_like(codes)
    scales = torch.empty(nb, device="cuda"); rscales = torch.empty_like(scales)
    bits = torch.zeros((nb + 31) // 32, dtype=torch.int32, device="cuda"); count = torch.zeros(1, dtype=torch.int32, device="cuda")
    x = bench.make_activations(R, C, 5, "cuda", torch.bfloat16)
    sc = fbq.score_blocks(x).cpu().numpy()
    theta, _ = fbq.theta_for_rate(sc, 0.0)
    for use_count in (True, False):
        def run():
            K.call("fbq_cuda_quantize_fallback", x.data_ptr(), K.FBQ_BF16, R, C, C, K.FBQ_MASK_THRESHOLD, theta,
                   bits.data_ptr(), codes.data_ptr(), C, scales.data_ptr(), res.data_ptr(), rscales.data_ptr(),
                   count.data_ptr() if use_count else None, None, None, 0, 0, stream.cuda_stream)
        for _ in range(3): run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(stream)
        for _ in range(20): run()
        e1.record(stream); torch.cuda.synchronize()
        print(R, C, "count" if use_count else "no count", round(e0.elapsed_time(e1) / 20 * 1e3, 1), "us", flush=True)

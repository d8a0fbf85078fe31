"""Where K1's fixed per-call cost on small shapes goes: host enqueue rate,
event-timed back-to-back calls, the same 20 calls replayed from a CUDA graph,
and a plain copy of the same bytes (torch copy_)."""
import sys, os, json, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2503_08040_b200 import fbq
from paper_2503_08040_b200 import _capi as K

peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
s = torch.cuda.Stream()
torch.cuda.set_stream(s)


def ev_time(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(s)
    for _ in range(n):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e-3


def graph_time(fn, n=20):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(n):
            fn()
    g.replay()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(s)
        g.replay()
        e1.record(s)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / n * 1e-3)
    return best


for dt in (torch.bfloat16, torch.float32):
    for (R, C) in [(2048, 4096), (4096, 4096), (8192, 4096), (16384, 4096), (8192, 14336)]:
        nb = (R // 128) * (C // 128)
        x = bench.make_activations(R, C, 5, "cuda", dt)
        codes = torch.empty(R, C, dtype=torch.int8, device="cuda")
        res = torch.empty_like(codes)
        scales = torch.empty(nb, device="cuda")
        rscales = torch.empty_like(scales)
        bits = torch.zeros((nb + 31) // 32, dtype=torch.int32, device="cuda")
        count = torch.zeros(1, dtype=torch.int32, device="cuda")
        theta = float(fbq.score_blocks(x).max().item()) * 2.0
        byt = R * C * (x.element_size() + 1)
        cp_src = torch.empty(byt // 4, dtype=torch.bfloat16, device="cuda")  # copy: reads + writes byt / 2 each
        cp_dst = torch.empty_like(cp_src)

        def k1():
            K.call("fbq_cuda_quantize_fallback", x.data_ptr(), K.FBQ_BF16 if dt == torch.bfloat16 else K.FBQ_F32,
                   R, C, C, K.FBQ_MASK_THRESHOLD, theta, bits.data_ptr(), codes.data_ptr(), C,
                   scales.data_ptr(), res.data_ptr(), rscales.data_ptr(), count.data_ptr(),
                   None, None, 0, 0, s.cuda_stream)

        def cp():
            cp_dst.copy_(cp_src)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(200):
            k1()
        host = (time.perf_counter() - t0) / 200
        torch.cuda.synchronize()
        tk, tg = ev_time(k1), graph_time(k1)
        tc, tcg = ev_time(cp), graph_time(cp)
        key = f"{R}x{C} {str(dt)[6:]}"
        r = {"MB": round(byt / 1e6, 1), "host_enqueue_us": round(host * 1e6, 2), "k1_events_us": round(tk * 1e6, 2),
             "k1_graph_us": round(tg * 1e6, 2), "copy_events_us": round(tc * 1e6, 2), "copy_graph_us": round(tcg * 1e6, 2),
             "k1_frac_events": round(byt / tk / 1e9 / peak, 3), "k1_frac_graph": round(byt / tg / 1e9 / peak, 3),
             "copy_frac_graph": round(byt / tcg / 1e9 / peak, 3)}
        print(key, r, flush=True)
        del x, codes, res, cp_src, cp_dst

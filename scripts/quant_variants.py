"""C2 bf16 sweep under K1 variants (diag 0: 1 stage x 4 CTAs, 2048: 2 x 3, 4: 3 x 2; 4096: static schedule)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2503_08040_b200 import fbq
lib = fbq.K.lib
lib.fbq_debug_set_quant_diag.argtypes = [fbq.K.cint]
peaks = json.load(open("MEASURED_PEAKS.json"))
for d in [int(a) for a in sys.argv[1:]] or [0, 2048, 4, 4096]:
    lib.fbq_debug_set_quant_diag(d)
    r = bench.quant_sweep("cuda", peaks.get("hbm_gbs", 6522.1))
    print("diag", d, {k: v["frac_hbm"] for k, v in r["cases"].items() if "bfloat16" in k}, flush=True)
lib.fbq_debug_set_quant_diag(0)

"""Run bench.py's C2 quantizer sweep alone (GB/s and HBM fraction per case)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
r = bench.quant_sweep("cuda", peaks.get("hbm_gbs", 6522.1))
for k, v in r["cases"].items():
    print(f"{k:32s} {v}")

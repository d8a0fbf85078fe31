"""bench.quant_sweep alone (C2, events + CUDA-graph timings + copy comparator), compact print."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
r = bench.quant_sweep("cuda", peak)
for k, v in r["cases"].items():
    print(f"{k:42s} us {v['us']:7.1f} frac {v['frac_hbm']:.3f}  graph {v['graph_us']:7.1f} {v['frac_hbm_graph']:.3f}"
          + (f"  flagged {v['flagged']:.3f}" if "flagged" in v else ""), flush=True)

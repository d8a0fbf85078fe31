"""Run selected bench.py parts alone: python scripts/bench_parts.py c4 exact ctx rms."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
parts = sys.argv[1:] or ["c4", "exact", "ctx", "rms"]
fns = {"c4": lambda: bench.qwen_block_linears("cuda"), "exact": lambda: bench.exact_mode_rate("cuda"),
       "ctx": lambda: bench.context_memory("cuda"), "rms": lambda: bench.rmsnorm_perf("cuda"),
       "c5": lambda: bench.c5_fallback_gemm("cuda"), "gemm": lambda: bench.gemm_sweep("cuda")}
for p in parts:
    print(p, json.dumps(fns[p]()), flush=True)

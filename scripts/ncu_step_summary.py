"""Summarise an `ncu --set full` capture of one MLP step (scripts/prof_kernels.py mlp)
into profiles/…_ncu_step_summary.json: per kernel launch the duration, DRAM bytes,
tensor/ALU/FMA pipe activity, issue activity, registers and occupancy."""
import csv, json, subprocess, sys

rep, dst = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, units = rows[0], rows[1]
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "sm__cycles_elapsed.avg.per_second"]
idx = {k: h.index(k) for k in keys if k in h}
out = {"source": f"ncu --set full --clock-control none ({rep}), one MLP fwd+bwd step, B200",
       "units": {k: units[i] for k, i in idx.items()}, "kernels": []}
for r in rows[2:]:
    d = {}
    for k, i in idx.items():
        v = r[i]
        try:
            d[k] = float(v.replace(",", ""))
        except ValueError:
            d[k] = v.split("(")[0].replace("void ", "").replace("fbq::", "")
    out["kernels"].append(d)
json.dump(out, open(dst, "w"), indent=1)
for d in out["kernels"]:
    print(f"{d['Kernel Name'][:48]:48s} {d.get('gpu__time_duration.sum', 0):9.3f} "
          f"dram {d.get('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 0):5.1f}% "
          f"tc {d.get('sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active', 0):5.1f}% "
          f"issue {d.get('sm__issue_active.avg.pct_of_peak_sustained_elapsed', 0):5.1f}%")

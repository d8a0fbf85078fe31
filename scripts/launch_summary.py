"""Summarise an ncu launch list (gpu__time_duration.sum per launch) of
`bench.py --steps 2 --warmup 1 --no-sweep` into per-kernel time and share of
the LAST step (the kernels after the last controller launch pair)."""
import csv, collections, json, sys

src, dst = sys.argv[1], sys.argv[2]
rows = [r for r in csv.reader(open(src)) if len(r) > 10]
h = rows[0]
ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
data = [(r[ki], float(r[vi].replace(",", ""))) for r in rows[1:] if r[mi] == "gpu__time_duration.sum"]
# a step ends with the two controller launches (gate/up, down)
ends = [i for i, (k, _) in enumerate(data) if "fbq_controller_kernel" in k]
last = data[ends[-4] + 1: ends[-1] + 1] if len(ends) >= 4 else data
agg = collections.defaultdict(lambda: [0, 0.0])
for k, v in last:
    name = k.split("(")[0].replace("void ", "").replace("fbq::", "")
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())
out = {"source": f"ncu --metrics gpu__time_duration.sum --clock-control none, bench.py --steps 2 --warmup 1 "
                 f"--no-sweep (last step's {len(last)} launches; cold-cache serialised: compare shares)",
       "step_us": round(tot / 1e3, 1),
       "kernels": [{"kernel": k, "launches": n, "us": round(t / 1e3, 1), "share": round(t / tot, 3)}
                   for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])]}
json.dump(out, open(dst, "w"), indent=1)
print(json.dumps(out, indent=1))

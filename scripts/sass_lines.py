"""Executed instructions per CUDA source line of one kernel: the ncu source page
(`ncu -i rep --page source --csv --print-source sass`) joined with nvdisasm's
line table (`nvdisasm -gi -c -fun <symbol index> <cubin>`; cubin from
`cuobjdump -xelf all lib.so`).  Lines are attributed to the outermost call
site inside the kernel.  usage: sass_lines.py ncu_sass.csv kernel.dis [top]"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
h, data = rows[1], rows[2:]
ai, ii = h.index("Address"), h.index("Instructions Executed")
ws = h.index("Warp Stall Sampling (All Samples)")
base = int(data[0][ai], 16)
cnt, stl = {}, {}
for r in data:
    try:
        off = int(r[ai], 16) - base
        cnt[off], stl[off] = int(r[ii]), int(r[ws] or 0)
    except ValueError:
        pass
cur, by, bys = None, collections.Counter(), collections.Counter()
for line in open(sys.argv[2]):
    m = re.search(r'//## File "[^"]+", line (\d+).*', line)
    if m:
        cur = re.findall(r"line (\d+)", m.group(0))[-1]
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", line)
    if m and cur:
        off = int(m.group(1), 16)
        by[cur] += cnt.get(off, 0)
        bys[cur] += stl.get(off, 0)
tot = sum(by.values())
print(f"executed warp instructions: {tot}")
for k, v in by.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 20):
    print(f"{v / tot * 100:5.1f} %  stall samples {bys[k]:6d}  line {k}")

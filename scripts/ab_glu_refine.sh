# A/B of two builds of the library in one gpurun call: A = lib/ (default build),
# B = ab/libfbq_b200.so (a variant built by hand, e.g. -DFBQ_CTX_REFINE=0), GLU forward
# kernel time under ncu for each, interleaved A B A B.
mkdir -p gpurun_out
for v in A B A B; do
  if [ $v = B ]; then export FBQ_B200_LIB_OVERRIDE=$PWD/ab/libfbq_b200.so; else unset FBQ_B200_LIB_OVERRIDE; fi
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"glu_forward" --csv --log-file gpurun_out/glf_$v.csv python scripts/mlp_ab.py 0 > /dev/null 2>&1
  python - $v <<PY
import csv,sys
rows=[r for r in csv.reader(open("gpurun_out/glf_"+sys.argv[1]+".csv")) if len(r)>10]
h=rows[0]; vi=h.index("Metric Value")
v=sorted(float(r[vi].replace(",","")) for r in rows[1:])
print(sys.argv[1], "refine" if sys.argv[1]=="A" else "no-refine", len(v), v[len(v)//2])
PY
done

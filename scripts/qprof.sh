# ncu --set full of the C2 quantizer (K1) at 8192x14336 bf16 0 / 5 %, 8192x4096 bf16 0 %, 8192x14336 fp32 5 %
set -x
mkdir -p gpurun_out
for c in "8192 14336 bf16 0.0" "8192 14336 bf16 0.05" "8192 4096 bf16 0.0" "8192 14336 f32 0.05"; do
  tag=$(echo $c | tr ' ' '_')
  ncu --set full --clock-control none --import-source on -k regex:quantize -s 2 -c 1 -o gpurun_out/q2_$tag python scripts/quant_prof.py $c > /dev/null 2>&1
done
ls gpurun_out

# compute-sanitizer racecheck (shared-memory hazards) and synccheck over small
# GPU tests of the kernels with CTA-level shared-memory protocols (K1 rings,
# RmsNorm cp.async rings, GLU staging, fused RmsNorm -> K1, SGD + RTN)
mkdir -p gpurun_out
out=gpurun_out/racecheck_r02.txt
echo "compute-sanitizer racecheck / synccheck, round 2 (B200)" > $out
run() {
  tool=$1; shift
  echo "--- $tool $*" >> $out
  timeout 1200 compute-sanitizer --tool $tool --print-limit 5 python -m pytest "$@" -q -x 2>&1 | grep -E "passed|failed|ERROR SUMMARY|hazard|Race|race|barrier" | head -8 >> $out
}
run racecheck tests/test_gpu_rmsnorm.py -k "384 or 512"
run racecheck tests/test_gpu_parity.py -k "dynamic_block_schedule"
run racecheck tests/test_gpu_sgd.py -k "matches_update"
run racecheck tests/test_gpu_mlp.py -k "step_bit_exact"
run racecheck tests/test_gpu_glublock.py -k "equals_norm"
run synccheck tests/test_gpu_rmsnorm.py -k "384 or 512"
run synccheck tests/test_gpu_parity.py -k "dynamic_block_schedule"
run synccheck tests/test_gpu_mlp.py -k "step_bit_exact"
cat $out

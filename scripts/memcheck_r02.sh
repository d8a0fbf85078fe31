# compute-sanitizer memcheck over the GPU tests touched in round 2 session 2
mkdir -p gpurun_out
out=gpurun_out/memcheck_r02.txt
echo "compute-sanitizer --tool memcheck, round 2 session 2 (B200)" > $out
run() {
  echo "--- $*" >> $out
  timeout 900 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest "$@" -q -x 2>&1 | grep -E "passed|failed|ERROR SUMMARY|Invalid|out of bounds" | head -8 >> $out
}
run tests/test_gpu_rmsnorm.py
run tests/test_gpu_parity.py -k "dynamic_block_schedule or threshold or given_mask or tile_rasters or gemm_fma"
run tests/test_gpu_rounding.py -k packed
run tests/test_gpu_mlp.py
run tests/test_gpu_linear.py
run tests/test_gpu_abi_contract.py
run tests/test_gpu_sgd.py
run tests/test_gpu_glublock.py
run tests/test_gpu_determinism.py -k repeatable
cat $out

#!/bin/bash
# GEMM change check: parity tests of the GEMM, role isolation, quick perf.
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "gemm or block_products" > gpurun_out/gemm_parity.log 2>&1; echo "rc=$?" >> gpurun_out/gemm_parity.log
tail -5 gpurun_out/gemm_parity.log
if grep -q "rc=0" gpurun_out/gemm_parity.log; then
  timeout 200 python scripts/gemm_isolate.py 0 1 ${ISO_DIAGS} > gpurun_out/gemm_iso.txt 2>&1; cat gpurun_out/gemm_iso.txt
  timeout 300 python scripts/quick_perf.py > gpurun_out/quick_perf.txt 2>&1; cat gpurun_out/quick_perf.txt
fi

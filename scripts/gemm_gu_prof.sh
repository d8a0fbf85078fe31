# ncu --set full of the dominant GEMM launch (gate/up forward) of the C3 step
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:fbq_gemm_kernel -s 7 -c 1 -o gpurun_out/r02s2_gemm_gu_full python scripts/prof_kernels.py mlp > gpurun_out/gemm_gu_prof.log 2>&1
tail -2 gpurun_out/gemm_gu_prof.log

# ncu --set full of the SR-heavy kernels of one MLP step (X quantizer, GLU fwd/bwd, SR(dY))
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"glu|quantize_block" -s 8 -c 4 -o gpurun_out/sr_kernels python scripts/mlp_one_step.py > gpurun_out/sr_prof.log 2>&1
tail -3 gpurun_out/sr_prof.log

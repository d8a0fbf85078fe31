mkdir -p gpurun_out
python scripts/dx_traffic.py 0 2097152 134217728 136314880
for d in 2097152 136314880; do
REPS=1 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemm -s 2 -c 1 python scripts/dx_traffic.py $d 2>&1 | grep -E "dram__|gpu__time"
done

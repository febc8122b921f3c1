CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --batch 0 --c4 0"
$CMD > gpurun_out/plain.log 2>&1 || exit 1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:'k_build|k_calibrate|k_register' --csv --log-file gpurun_out/dram2.csv $CMD > /dev/null 2>&1
grep -E "k_build" gpurun_out/dram2.csv | head -6

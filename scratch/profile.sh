#!/bin/bash
# Round profile: launch list, DRAM bytes of the build kernels, and one full
# capture of each persistent kernel (each ncu run only after the same command
# exited 0 without ncu).
set -x
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --batch 0 --c4 0"
$CMD > gpurun_out/plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:'k_build|k_calibrate|k_register' --csv --log-file gpurun_out/dram.csv $CMD > gpurun_out/ncu_dram.log 2>&1
for K in k_build k_calibrate k_register; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s 0 -c 1 -o gpurun_out/prof_$K -f $CMD > gpurun_out/ncu_$K.log 2>&1
done
ls -la gpurun_out

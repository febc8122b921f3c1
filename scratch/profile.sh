#!/bin/bash
# Round profile: launch list + one full capture of each persistent kernel.
set -x
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_build -s 0 -c 1 -o gpurun_out/prof_build $CMD > gpurun_out/ncu_build.log 2>&1
$CMD > gpurun_out/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_register -s 0 -c 1 -o gpurun_out/prof_register $CMD > gpurun_out/ncu_register.log 2>&1
ls -la gpurun_out

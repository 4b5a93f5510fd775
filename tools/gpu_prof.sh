#!/usr/bin/env bash
# Full ncu capture of k_wbm launches (negative + positive phase of one step) and the step's launch list.
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_wbm -s ${SKIP:-6} -c ${COUNT:-2} \
    -o gpurun_out/prof_wbm python bench.py --steps 1 --warmup 4 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
tail -2 gpurun_out/ncu_full.log

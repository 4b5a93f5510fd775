#!/usr/bin/env bash
# C4 launch list (one timed step) and a full capture of the merge kernels of one batch.
mkdir -p gpurun_out
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/launches_c4.csv -k regex:'^k_' \
    python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c4_launch.log 2>&1
echo "launch rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'k_merge|k_alloc' -s ${SKIP:-9} -c 4 \
    -o gpurun_out/prof_c4_merge python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c4_full.log 2>&1
echo "full rc=$?"
tail -2 gpurun_out/ncu_c4_full.log

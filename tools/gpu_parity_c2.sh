#!/usr/bin/env bash
# C2 bench line with full-batch parity against the restatement (all 8 batches).
mkdir -p gpurun_out
make -s -C oracle
df -h /tmp > gpurun_out/df.txt 2>&1
timeout 1500 python bench.py --steps 5 --warmup 3 --cpu-batches 2 > gpurun_out/bench_pf.json 2> gpurun_out/bench_pf.log
tail -5 gpurun_out/bench_pf.log

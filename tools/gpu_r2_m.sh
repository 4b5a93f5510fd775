#!/usr/bin/env bash
# Round 2, call M: C5 batch-size sweep (1K..1M, exact coalescing), 1-GPU shard simulations of C2 and C4 (stream).
mkdir -p gpurun_out/m
O=gpurun_out/m/sweep T=1500 bash tools/gpu_sweep_c5.sh > gpurun_out/m/sweep.txt 2>&1
timeout 1200 python tools/shard_sim.py --config C2 --worlds 1,2,4,8 --steps 5 --out gpurun_out/m/shard_c2.json > gpurun_out/m/shard_c2.log 2>&1
timeout 2400 python tools/shard_sim.py --config C4 --worlds 1,2,4,8 --steps 3 --out gpurun_out/m/shard_c4.json > gpurun_out/m/shard_c4.log 2>&1
cat gpurun_out/m/sweep.txt; tail -4 gpurun_out/m/shard_c2.log; tail -4 gpurun_out/m/shard_c4.log
O=gpurun_out/m/cli bash tools/cli_pipeline.sh > gpurun_out/m/cli.txt 2>&1; cat gpurun_out/m/cli.txt
# repeated A/B of the throughput variant on C4 (alternating)
for i in 1 2; do for v in 3 4; do
  BDSM_TUNE_VARIANT_THROUGHPUT=$v timeout 900 python bench.py --config C4 --steps 4 --warmup 3 --no-cpu-baseline --parity-full 0 > gpurun_out/m/c4_v${v}_$i.json 2> gpurun_out/m/c4_v${v}_$i.log
  python -c "import json,sys; d=json.loads(open('gpurun_out/m/c4_v${v}_$i.json').read().strip().splitlines()[-1]); print('c4 v$v run $i', d['value'], d['ms_per_step'])"
done; done

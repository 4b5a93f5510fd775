#!/usr/bin/env bash
# Round 2, call K: A/B of the shared-memory staging (default build vs -DBDSM_NO_STAGE) on C2, test durations.
mkdir -p gpurun_out/k
O=gpurun_out/k
NS=$PWD/paper_2401_17018_b200/libbdsm_b200_nostage.so
for r in 1 2; do
  timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --parity-full 0 > $O/stage_$r.json 2> $O/stage_$r.log
  BDSM_LIB=$NS timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --parity-full 0 > $O/nostage_$r.json 2> $O/nostage_$r.log
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q --durations=8 > $O/durations.log 2>&1
BDSM_LIB=$NS timeout 900 python -m pytest tests/test_gpu_parity.py -q --durations=8 > $O/durations_nostage.log 2>&1
for f in $O/*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']/1e6,3), round(d['ms_per_step'],4), round(d['latency']['ms_per_batch'],4))"; done
tail -12 $O/durations.log; tail -12 $O/durations_nostage.log

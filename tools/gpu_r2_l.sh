#!/usr/bin/env bash
# Round 2, call L: matching-kernel variant A/B on the throughput configs (4 CTAs/SM with spills vs 3 without),
# C2 recheck, CLI pipeline overlap measurement.
mkdir -p gpurun_out/l
O=gpurun_out/l
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --parity-full 0 > $O/c2.json 2> $O/c2.log
for v in 4 3; do
  BDSM_TUNE_VARIANT_THROUGHPUT=$v timeout 900 python bench.py --config C4 --steps 4 --warmup 3 --no-cpu-baseline > $O/c4_v$v.json 2> $O/c4_v$v.log
  BDSM_TUNE_VARIANT_THROUGHPUT=$v timeout 900 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline --parity-full 0 --coalesce > $O/c5_v$v.json 2> $O/c5_v$v.log
  BDSM_TUNE_VARIANT_THROUGHPUT=$v timeout 900 python bench.py --config C3 --batch 20000 --steps 3 --warmup 3 --no-cpu-baseline --parity-full 0 > $O/c3_v$v.json 2> $O/c3_v$v.log
done
O=$O/cli timeout 1200 bash tools/cli_pipeline.sh > gpurun_out/l/cli.txt 2>&1
for f in gpurun_out/l/*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d.get('value'), d.get('ms_per_step'))" 2>/dev/null || echo "$f failed"; done
cat gpurun_out/l/cli.txt

#!/usr/bin/env bash
# Parity tests + bench lines for every config (no CPU baseline).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
for c in ${CONFIGS:-C2 C1 C3 C5 C5cycle}; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.log
  echo "$c rc=$?"; python -c "
import json,sys
try:
  b=json.load(open('gpurun_out/bench_$c.json'))
  print('  value %.0f e2e %.0f ms/step %.3f frac %.3f parity %s' % (b['value'], b['e2e']['value'], b['ms_per_step'], b['roofline']['frac'], b['counts']['e2e_equals_device_path']))
  print('  per-step ms', [round(s['ms'],3) for s in b['per_step']])
except Exception as e: print('  failed', e); print(open('gpurun_out/bench_$c.log').read()[-1500:])
"
done

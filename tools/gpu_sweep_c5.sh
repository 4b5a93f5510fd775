#!/usr/bin/env bash
# C5: batch-size sweep with the unlabelled 5-clique and 5-cycle queries (BASELINE configs[4]).
mkdir -p gpurun_out
for cfg in C5 C5cycle; do
  for bs in ${SIZES:-1000 10000 100000}; do
    if [ "$cfg" = C5cycle ] && [ "$bs" -gt 10000 ]; then continue; fi
    timeout 900 python bench.py --config $cfg --batch $bs --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/sweep_${cfg}_$bs.json 2>/dev/null
    python -c "
import json
b=json.load(open('gpurun_out/sweep_${cfg}_$bs.json'))
print('$cfg', $bs, 'updates/s %.0f' % b['value'], 'e2e %.0f' % b['e2e']['value'], 'ms/step %.2f' % b['ms_per_step'],
      'neg', b['counts']['negative'][-1], 'pos', b['counts']['positive'][-1])" || echo "$cfg $bs failed"
  done
done

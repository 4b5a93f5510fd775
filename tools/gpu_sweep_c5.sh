#!/usr/bin/env bash
# C5: batch-size sweep 1K..1M with the unlabelled 5-clique and 5-cycle queries (BASELINE configs[4]),
# exact coalescing on (counts equal coalesce off); restatement parity on the smaller sizes.
O=${O:-gpurun_out/sweep}
mkdir -p $O
for cfg in C5 C5cycle; do
  for bs in ${SIZES:-1000 10000 100000 1000000}; do
    pf=0
    if [ "$cfg" = C5 ] && [ "$bs" -le 10000 ]; then pf=-1; fi
    steps=3
    if [ "$bs" -ge 1000000 ]; then steps=2; fi
    timeout ${T:-1200} python bench.py --config $cfg --batch $bs --steps $steps --warmup 3 --no-cpu-baseline \
        --parity-full $pf --coalesce > $O/sweep_${cfg}_$bs.json 2> $O/sweep_${cfg}_$bs.log
    python -c "
import json
b=json.loads(open('$O/sweep_${cfg}_$bs.json').read().strip().splitlines()[-1])
print('$cfg', $bs, 'updates/s %.0f' % b['value'], 'e2e %.0f' % b['e2e']['value'], 'ms/step %.2f' % b['ms_per_step'],
      'neg', b['counts']['negative'][-1], 'pos', b['counts']['positive'][-1], 'parity', (b.get('parity_full') or {}).get('equal'))" || echo "$cfg $bs failed"
  done
done

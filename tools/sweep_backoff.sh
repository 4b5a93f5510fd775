#!/usr/bin/env bash
# Idle-warp backoff sweep (BDSM_TUNE_BACKOFF, ns) on C2, 12 steps each.
for b in ${BACKOFFS:-256 512 1024 2048}; do
  r=$(BDSM_TUNE_BACKOFF=$b timeout 600 python bench.py --steps 12 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; b=json.load(sys.stdin); print(round(b['value']), round(b['ms_per_step'],4), 'neg', round(sum(s['neg_ms'] for s in b['per_step']),3), 'pos', round(sum(s['pos_ms'] for s in b['per_step']),3))")
  echo "backoff $b: $r"
done

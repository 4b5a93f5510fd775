#!/usr/bin/env bash
# Idle-warp backoff on the throughput configs (C4, C5, C3).
for c in ${CFGS:-C4 C5 C3}; do for b in 256 1024; do
  r=$(BDSM_TUNE_BACKOFF=$b timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; b=json.load(sys.stdin); print(round(b['value']), round(b['ms_per_step'],3))")
  echo "$c backoff $b: $r"
done; done

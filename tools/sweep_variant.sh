#!/usr/bin/env bash
# Matching-kernel variant (CTAs per SM) sweep on C2 and C5.
for v in 2 3 4; do
  r=$(BDSM_TUNE_VARIANT=$v timeout 600 python bench.py --steps 12 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; b=json.load(sys.stdin); print(round(b['value']), round(b['ms_per_step'],4), [round(s['neg_ms'],3) for s in b['per_step']])")
  echo "C2 variant $v: $r"
done
for v in 3 4; do
  r=$(BDSM_TUNE_VARIANT=$v timeout 900 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; b=json.load(sys.stdin); print(round(b['value']), round(b['ms_per_step'],3))")
  echo "C5 variant $v: $r"
done

#!/usr/bin/env bash
# C4 (and C2) merge time per list-length variant library (libbdsm_var_*.so).
for v in ${VARIANTS:-default B C D E}; do
  lib=paper_2401_17018_b200/libbdsm_b200.so
  [ "$v" != default ] && lib=paper_2401_17018_b200/libbdsm_var_$v.so
  r=$(BDSM_LIB=$PWD/$lib timeout 900 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; b=json.load(sys.stdin); print(round(b['value']), round(b['ms_per_step'],3), 'merge', [round(s['merge_ms'],3) for s in b['per_step']], b['counts']['e2e_equals_device_path'])")
  echo "C4 $v: $r"
  r=$(BDSM_LIB=$PWD/$lib timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; b=json.load(sys.stdin); print(round(b['value']), round(b['ms_per_step'],4), 'merge', [round(s['merge_ms'],3) for s in b['per_step']])")
  echo "C2 $v: $r"
done

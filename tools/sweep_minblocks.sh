#!/usr/bin/env bash
# Builds k_wbm with different register budgets (resident CTAs per SM) and benches each (GPU box).
for mb in ${MBS:-2 3 4}; do
  BDSM_NVCC_EXTRA="-DBDSM_WBM_MIN_BLOCKS=$mb" BDSM_OBJ=/tmp/obj_mb$mb BDSM_OUT=/tmp/libbdsm_mb$mb.so \
    bash paper_2401_17018_b200/build.sh > /tmp/build_mb$mb.log 2>&1 || { echo "build $mb failed"; continue; }
  grep -A2 "k_wbmILb0" /tmp/obj_mb$mb/match.ptxas.log | grep -E "registers" | head -1
  for rep in 1 2; do
    BDSM_LIB=/tmp/libbdsm_mb$mb.so python bench.py --steps 8 --warmup 3 --no-cpu-baseline 2>/dev/null | \
      python -c "import json,sys; b=json.load(sys.stdin); print('minblocks $mb', round(b['value']), round(b['ms_per_step'],3))"
  done
done

#!/usr/bin/env bash
# GPU-box helper: rebuild the engine with different register budgets for k_wbm
# and run the C2 bench for each (tuning experiment).
set -u
for mb in ${MINBS:-4 5 6 8}; do
  BDSM_NVCC_EXTRA="-DBDSM_WBM_MIN_BLOCKS=$mb" bash paper_2401_17018_b200/build.sh > /dev/null 2>&1
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null > gpurun_out/sweep_$mb.json
  python -c "
import json; d=json.load(open('gpurun_out/sweep_$mb.json')); print('minb=$mb', round(d['value']), [round(s['ms'],1) for s in d['per_step']])"
done
bash paper_2401_17018_b200/build.sh > /dev/null 2>&1

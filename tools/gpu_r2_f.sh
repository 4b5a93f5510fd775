#!/usr/bin/env bash
# Round 2, call F: full ncu capture (source-level) of a fused k_wbm launch (pos(i)+neg(i+1)) of a timed C2 stream,
# and of the single-phase negative launch of the per-batch path for comparison.
mkdir -p gpurun_out/f
O=gpurun_out/f
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k "regex:k_wbmILb0ELi2ELi2E" -s 4 -c 1 \
   -o $O/prof_fused python bench.py --steps 2 --warmup 3 --no-cpu-baseline --parity-full 0 > $O/ncu_fused.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k "regex:k_wbmILb0ELi2ELi1E" -s 6 -c 1 \
   -o $O/prof_single python bench.py --steps 1 --warmup 4 --no-cpu-baseline --parity-full 0 --no-stream > $O/ncu_single.log 2>&1
ls -la $O

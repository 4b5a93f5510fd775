#!/usr/bin/env bash
# Round 2: C3 matching-kernel variant for launches with many items (3 vs 4 CTAs/SM) and C1 short-list merge on/off,
# alternating variants on one workload each (tools/ab_env.py).
O=gpurun_out/ab2; mkdir -p $O
timeout 1200 python tools/ab_env.py --config C3 --steps 3 --warmup 3 --rounds 2 \
  --variant tp3: --variant tp4:BDSM_TUNE_VARIANT_THROUGHPUT=4 > $O/c3.txt 2> $O/c3.log
tail -2 $O/c3.txt
timeout 600 python tools/ab_env.py --config C1 --steps 10 --warmup 3 --rounds 3 \
  --variant base: --variant nosmall:BDSM_TUNE_SMALLMIN=65536 > $O/c1.txt 2> $O/c1.log
tail -2 $O/c1.txt

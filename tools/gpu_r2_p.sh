#!/usr/bin/env bash
# Round 2, call P: list-length thresholds of the merge kernels (tools/ab_env.py, one workload per config,
# variants alternating), after the short-list kernel choice by batch size.
mkdir -p gpurun_out/p
timeout 1500 python tools/ab_env.py --config C4 --steps 4 --warmup 3 --rounds 2 \
  --variant big1024: --variant big2048:BDSM_TUNE_BIGLIST_LARGE=2048 --variant big4096:BDSM_TUNE_BIGLIST_LARGE=4096 \
  --variant big512:BDSM_TUNE_BIGLIST_LARGE=512 > gpurun_out/p/c4.txt 2> gpurun_out/p/c4.log
tail -5 gpurun_out/p/c4.txt
timeout 900 python tools/ab_env.py --config C2 --steps 10 --warmup 3 --rounds 3 \
  --variant base: --variant big512:BDSM_TUNE_BIGLIST=512 --variant big2048:BDSM_TUNE_BIGLIST=2048 \
  --variant smax512:BDSM_TUNE_SMALLMAX=512 --variant smax128:BDSM_TUNE_SMALLMAX=128 --variant g16:BDSM_TUNE_SMALL_GROUP=16 \
  --variant nosmall:BDSM_TUNE_SMALLMIN=65536 > gpurun_out/p/c2.txt 2> gpurun_out/p/c2.log
tail -8 gpurun_out/p/c2.txt

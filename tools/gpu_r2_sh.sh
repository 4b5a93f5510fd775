#!/usr/bin/env bash
# Round 2: shard simulation with the final build (C2 at 1/2/4/8 ranks, C4 at 1/8).
O=gpurun_out/sh; mkdir -p $O
timeout 900 python tools/shard_sim.py --config C2 --worlds 1,2,4,8 --steps 5 --out $O/shard_c2.json > $O/shard_c2.log 2>&1
timeout 1200 python tools/shard_sim.py --config C4 --worlds 1,8 --steps 3 --out $O/shard_c4.json > $O/shard_c4.log 2>&1
grep "W=" $O/shard_c2.log $O/shard_c4.log

#!/usr/bin/env bash
# Round 2, call V: contiguous per-rank work-item ranges — shard/group tests, then the shard simulation of C4 / C2.
O=gpurun_out/v; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_group.py tests/test_gpu_parity.py -m gpu -x -q -k "group or split or shard" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
tail -3 $O/pytest.log
timeout 2400 python tools/shard_sim.py --config C4 --worlds 1,2,8 --steps 3 --out $O/shard_c4.json > $O/shard_c4.log 2>&1
grep "W=" $O/shard_c4.log
timeout 1200 python tools/shard_sim.py --config C2 --worlds 1,2,4,8 --steps 5 --out $O/shard_c2.json > $O/shard_c2.log 2>&1
grep "W=" $O/shard_c2.log

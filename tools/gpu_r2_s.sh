#!/usr/bin/env bash
# Round 2, call S: multi-device group (bdsm_group_*: C ABI, ctypes, CLI --devices) on the one GPU, then the
# 1-GPU shard simulation of C2 and C4 with the current merge kernels.
O=gpurun_out/s; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_group.py tests/test_cli.py -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
tail -3 $O/pytest.log
timeout 1200 python tools/shard_sim.py --config C2 --worlds 1,2,4,8 --steps 5 --out $O/shard_c2.json > $O/shard_c2.log 2>&1
tail -6 $O/shard_c2.log
timeout 2400 python tools/shard_sim.py --config C4 --worlds 1,2,8 --steps 3 --out $O/shard_c4.json > $O/shard_c4.log 2>&1
tail -6 $O/shard_c4.log

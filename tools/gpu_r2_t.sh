#!/usr/bin/env bash
# Round 2, call T: one-wave merge grids, 16-entry run copies and the label index without a local array —
# short-list and stream parity tests, then C4 and C2 bench lines.
O=gpurun_out/t; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stream.py tests/test_gpu_scale.py -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
tail -3 $O/pytest.log
timeout 900 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline --parity-full 0 > $O/c4.json 2> $O/c4.log
python tools/bench_brief.py $O/c4.json c4
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --parity-full 0 > $O/c2.json 2> $O/c2.log
python tools/bench_brief.py $O/c2.json c2
timeout 900 python tools/ab_env.py --config C4 --steps 4 --warmup 3 --rounds 2 \
  --variant base: --variant big2048:BDSM_TUNE_BIGLIST_LARGE=2048 --variant smax128:BDSM_TUNE_SMALLMAX=128 > $O/ab_c4.txt 2> $O/ab_c4.log
tail -3 $O/ab_c4.txt

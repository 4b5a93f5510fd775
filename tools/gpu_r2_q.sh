#!/usr/bin/env bash
# Round 2, call Q: CTA-aggregated k_alloc, unpredicated run copies, barrier-free column-size flush —
# GPU parity suites, then C4 / C2 A/B of the short-list and long-list choices on the new build.
mkdir -p gpurun_out/q
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/q/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q/pytest.log
tail -3 gpurun_out/q/pytest.log
timeout 1500 python tools/ab_env.py --config C4 --steps 4 --warmup 3 --rounds 2 \
  --variant base: --variant g8:BDSM_TUNE_SMALL_GROUP_LARGE=8 --variant big4096:BDSM_TUNE_BIGLIST_LARGE=4096 \
  > gpurun_out/q/c4.txt 2> gpurun_out/q/c4.log
tail -4 gpurun_out/q/c4.txt
timeout 900 python bench.py --config C4 --steps 4 --warmup 3 --no-cpu-baseline --parity-full 0 > gpurun_out/q/c4_bench.json 2> gpurun_out/q/c4_bench.log
python tools/bench_brief.py gpurun_out/q/c4_bench.json c4
timeout 900 python bench.py > gpurun_out/q/c2_bench.json 2> gpurun_out/q/c2_bench.log
python tools/bench_brief.py gpurun_out/q/c2_bench.json c2

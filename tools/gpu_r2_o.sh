#!/usr/bin/env bash
# Round 2, call O: the lane-group short-list merge (k_merge_group) — parity test over the
# short-list modes, then C4 A/B (group 8 / 16 / thread per list) and C2 with the short-list path on.
mkdir -p gpurun_out/o
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k thread_merge > gpurun_out/o/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/o/pytest.log
tail -3 gpurun_out/o/pytest.log
for v in 8 1 16; do
  BDSM_TUNE_SMALL_GROUP=$v timeout 900 python bench.py --config C4 --steps 4 --warmup 3 --no-cpu-baseline --parity-full 0 > gpurun_out/o/c4_g$v.json 2> gpurun_out/o/c4_g$v.log
  python tools/bench_brief.py gpurun_out/o/c4_g$v.json "c4 group $v"
done
for mn in 65536 1; do
  BDSM_TUNE_SMALLMIN=$mn timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --parity-full 0 > gpurun_out/o/c2_min$mn.json 2> gpurun_out/o/c2_min$mn.log
  python tools/bench_brief.py gpurun_out/o/c2_min$mn.json "c2 smallmin $mn"
done

#!/usr/bin/env bash
# One GPU session: parity tests, bench line (with CPU baseline), reference arm,
# launch list, full capture of the negative-phase k_wbm launch of a timed step.
set -x
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_wbm -s 6 -c 2 -o gpurun_out/prof_wbm \
    python bench.py --steps 1 --warmup 4 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_merge_refresh -s 3 -c 1 -o gpurun_out/prof_merge \
    python bench.py --steps 1 --warmup 4 --no-cpu-baseline > gpurun_out/ncu_merge.log 2>&1
ls -la gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log

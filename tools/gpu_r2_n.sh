#!/usr/bin/env bash
# Round 2, call N: HEAD check after the container restore (GPU tests, smoke, default bench line),
# then a full capture of the C4 short-list merge (k_merge_small) for its rewrite.
mkdir -p gpurun_out/n
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/n/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/n/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/n/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/n/smoke.log
timeout 900 python bench.py > gpurun_out/n/bench.json 2> gpurun_out/n/bench.log
tail -2 gpurun_out/n/pytest_gpu.log; tail -1 gpurun_out/n/smoke.log; cat gpurun_out/n/bench.json
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'k_merge_small' -s 3 -c 1 \
    -o gpurun_out/n/prof_c4_small python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline --parity-full 0 > gpurun_out/n/ncu_c4_small.log 2>&1
echo "ncu rc=$?"

#!/usr/bin/env bash
# Round-2 first confirmation: GPU tests, smoke, default bench line, launch list.
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/smi.txt 2>&1; nproc >> gpurun_out/smi.txt; lscpu | grep -i 'model name' >> gpurun_out/smi.txt; free -g >> gpurun_out/smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 5 --warmup 3 --cpu-batches 2 > gpurun_out/bench.json 2> gpurun_out/bench.log
tail -3 gpurun_out/pytest_gpu.log

#!/usr/bin/env bash
# GPU tests + parity at scale (C2 20 batches, C5 cycle, C3 prefixes, C4 prefix) with pruned-visit checks.
mkdir -p gpurun_out/parity
make -s -C oracle
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
run() { name=$1; shift; timeout ${T:-900} python tools/parity_scale.py "$@" --out gpurun_out/parity/$name.json > gpurun_out/parity/$name.log 2>&1; echo "$name rc=$?" >> gpurun_out/parity/summary.txt; }
run c2_full20 --config C2 --batches 20
run c5cycle_1k --config C5cycle --batches 2 --batch 1000
run c3_p1000 --config C3 --batches 3 --prefix 1000
run c3_p3000 --config C3 --batches 2 --prefix 3000
T=2400 run c4_p1000 --config C4 --batches 2 --prefix 1000
cat gpurun_out/parity/summary.txt; tail -3 gpurun_out/pytest_gpu.log

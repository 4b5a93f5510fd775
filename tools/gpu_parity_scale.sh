#!/usr/bin/env bash
# Parity at scale: CUDA engine vs the reference-pinned restatement on C1/C2/C3/C5.
mkdir -p gpurun_out/parity
make -s -C oracle
run() { name=$1; shift; timeout ${T:-900} python tools/parity_scale.py "$@" --out gpurun_out/parity/$name.json > gpurun_out/parity/$name.log 2>&1; echo "$name rc=$?" >> gpurun_out/parity/summary.txt; }
run c2_full --config C2 --batches 8
run c1_full --config C1 --batches 5
run c5clique_1k --config C5 --batches 3 --batch 1000
run c5cycle_1k --config C5cycle --batches 2 --batch 1000
run c3_p100 --config C3 --batches 3 --prefix 100
cat gpurun_out/parity/summary.txt

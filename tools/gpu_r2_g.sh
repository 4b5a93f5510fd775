#!/usr/bin/env bash
# Round 2, call G: stream tests + full GPU tests, default bench, 20-step bench.
mkdir -p gpurun_out/g
O=gpurun_out/g
make -s -C oracle
timeout 600 python -m pytest tests/test_gpu_stream.py -x -q > $O/pytest_stream.log 2>&1; echo "rc=$?" >> $O/pytest_stream.log
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 --cpu-batches 2 > $O/bench.json 2> $O/bench.log
timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --parity-full 0 > $O/bench_20.json 2> $O/bench_20.log
tail -3 $O/pytest_stream.log; tail -3 $O/pytest_gpu.log

#!/usr/bin/env bash
# Round 2, call H: stream tests + full GPU tests, C2 bench, then C1/C3/C4/C5 lines (stream where the graph exceeds L2).
mkdir -p gpurun_out/h
O=gpurun_out/h
make -s -C oracle
timeout 600 python -m pytest tests/test_gpu_stream.py -x -q > $O/pytest_stream.log 2>&1; echo "rc=$?" >> $O/pytest_stream.log
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 --cpu-batches 2 > $O/bench.json 2> $O/bench.log
timeout 900 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > $O/c4.json 2> $O/c4.log
timeout 900 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu-baseline --parity-full 0 > $O/c3.json 2> $O/c3.log
timeout 600 python bench.py --config C1 --steps 5 --warmup 3 --no-cpu-baseline > $O/c1.json 2> $O/c1.log
timeout 600 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline --coalesce > $O/c5.json 2> $O/c5.log
timeout 900 python bench.py --config C5cycle --steps 3 --warmup 3 --no-cpu-baseline --parity-full 0 --coalesce > $O/c5cyc.json 2> $O/c5cyc.log
tail -3 $O/pytest_stream.log; tail -3 $O/pytest_gpu.log

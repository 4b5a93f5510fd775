#!/usr/bin/env bash
# Round 2, call E: stream tests, full GPU tests, default bench, 20-step bench, traffic capture of the stream.
mkdir -p gpurun_out/e
O=gpurun_out/e
make -s -C oracle
timeout 600 python -m pytest tests/test_gpu_stream.py -x -q > $O/pytest_stream.log 2>&1; echo "rc=$?" >> $O/pytest_stream.log
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 --cpu-batches 2 > $O/bench.json 2> $O/bench.log
timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --parity-full 0 > $O/bench_20.json 2> $O/bench_20.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum \
   --clock-control none --csv --log-file $O/traffic_c2.csv \
   python bench.py --steps 5 --warmup 3 --no-cpu-baseline --parity-full 0 > $O/ncu_traffic.log 2>&1
python tools/ncu_traffic.py $O/traffic_c2.csv --steps 5 --wbm-per-step 1 --build $(python -c "import bench; print(bench.so_sha())" 2>/dev/null) --out $O/traffic_c2.json > /dev/null 2>&1
tail -3 $O/pytest_stream.log; tail -3 $O/pytest_gpu.log

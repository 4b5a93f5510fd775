#!/usr/bin/env bash
# Round 2, call J: staging + shared column-size aggregation: tests, racecheck, C2/C4 bench, C4 traffic of our kernels.
mkdir -p gpurun_out/j
O=gpurun_out/j
make -s -C oracle
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 --cpu-batches 2 > $O/bench.json 2> $O/bench.log
timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --parity-full 0 > $O/bench_20.json 2> $O/bench_20.log
timeout 900 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > $O/c4.json 2> $O/c4.log
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_golden.py fig1 skewed > $O/racecheck.log 2>&1; echo "rc=$?" >> $O/racecheck.log
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum \
   --clock-control none -k regex:"k_|Device" --csv --log-file $O/traffic_c4.csv \
   python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_c4.log 2>&1
python tools/ncu_traffic.py $O/traffic_c4.csv --steps 3 --wbm-per-step 1 --build $(python -c "import bench; print(bench.so_sha())" 2>/dev/null) --out $O/traffic_c4.json > /dev/null 2>&1
rm -f $O/traffic_c4.csv
tail -3 $O/pytest_gpu.log; tail -3 $O/racecheck.log

#!/usr/bin/env bash
# Round 2, call I: memo-bit filter check (tests), C2 + C4 bench, C4 traffic capture, sanitizers on golden suites.
mkdir -p gpurun_out/i
O=gpurun_out/i
make -s -C oracle
timeout 600 python -m pytest tests/test_gpu_stream.py tests/test_gpu_parity.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 --cpu-batches 2 > $O/bench.json 2> $O/bench.log
timeout 900 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > $O/c4.json 2> $O/c4.log
timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum \
   --clock-control none --csv --log-file $O/traffic_c4.csv \
   python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_c4.log 2>&1
python tools/ncu_traffic.py $O/traffic_c4.csv --steps 3 --wbm-per-step 1 --build $(python -c "import bench; print(bench.so_sha())" 2>/dev/null) --out $O/traffic_c4.json > /dev/null 2>&1
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_golden.py fig1 skewed matcher_random > $O/memcheck.log 2>&1; echo "rc=$?" >> $O/memcheck.log
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_golden.py fig1 skewed > $O/racecheck.log 2>&1; echo "rc=$?" >> $O/racecheck.log
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_golden.py fig1 > $O/synccheck.log 2>&1; echo "rc=$?" >> $O/synccheck.log
rm -f $O/traffic_c4.csv
tail -3 $O/pytest.log; tail -3 $O/memcheck.log; tail -3 $O/racecheck.log

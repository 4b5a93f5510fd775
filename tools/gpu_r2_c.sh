#!/usr/bin/env bash
# Round 2, call C: GPU tests; default bench (parity_full); ncu traffic capture -> profiles json;
# shard simulation C2; 2-rank spawn; C5 coalesce on/off; C2 trace diagnostics.
mkdir -p gpurun_out/c
O=gpurun_out/c
make -s -C oracle
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 --cpu-batches 2 > $O/bench.json 2> $O/bench.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum \
   --clock-control none --csv --log-file $O/traffic_c2.csv \
   python bench.py --steps 3 --warmup 3 --no-cpu-baseline --parity-full 0 > $O/ncu_traffic.log 2>&1
python tools/ncu_traffic.py $O/traffic_c2.csv --steps 3 --build $(python -c "import bench; print(bench.so_sha())" 2>/dev/null) --out $O/traffic_c2.json > /dev/null 2>&1
timeout 900 python tools/shard_sim.py --config C2 --worlds 1,2,4,8 --steps 3 --out $O/shard_c2.json > $O/shard_c2.log 2>&1
timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline --parity-full 0 > $O/bench_g2.json 2> $O/bench_g2.log
timeout 900 python bench.py --config C5 --batch 1000 --steps 5 --warmup 3 --no-cpu-baseline --parity-full 3 > $O/c5_off.json 2> $O/c5_off.log
timeout 900 python bench.py --config C5 --batch 1000 --steps 5 --warmup 3 --no-cpu-baseline --parity-full 3 --coalesce > $O/c5_on.json 2> $O/c5_on.log
timeout 900 python bench.py --config C5cycle --batch 1000 --steps 3 --warmup 3 --no-cpu-baseline --parity-full 0 --coalesce > $O/c5cyc_on.json 2> $O/c5cyc_on.log
BDSM_LIB=$PWD/paper_2401_17018_b200/libbdsm_b200_trace.so timeout 600 python tools/diag_c2.py --batches 8 --chunk 32 > $O/diag.txt 2>&1
tail -3 $O/pytest_gpu.log

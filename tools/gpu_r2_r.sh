#!/usr/bin/env bash
# Round 2, call R: C4 per-kernel traffic of the current build (metrics pass over 3 stream steps) and full
# captures of the merge kernels and k_validate of one batch.
O=gpurun_out/r; mkdir -p $O
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum \
   --clock-control none -k regex:"k_|Device" --csv --log-file $O/traffic_c4.csv \
   python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline --parity-full 0 > $O/ncu_c4.log 2>&1
echo "metrics rc=$?"
python tools/ncu_traffic.py $O/traffic_c4.csv --steps 3 --wbm-per-step 1 --build $(python -c "import bench; print(bench.so_sha())" 2>/dev/null) --out $O/traffic_c4.json
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:'k_merge_small|k_merge_refresh|k_alloc|k_validate|k_merge_big' -s 15 -c 5 \
    -o $O/prof_c4_merge python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline --parity-full 0 > $O/ncu_c4_full.log 2>&1
echo "full rc=$?"

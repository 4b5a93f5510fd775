#!/usr/bin/env bash
# Round 2, last call: matching-kernel variant by items per phase (4 CTAs/SM for mid-size launches such as C3, 3 for
# the largest such as C4).  Same-build traffic captures first, then GPU tests, smoke, C2 / C4 / C3 lines.
O=gpurun_out/zz; mkdir -p $O
SHA=$(python -c "import bench; print(bench.so_sha())" 2>/dev/null)
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum \
   --clock-control none -k regex:"k_|Device" --csv --log-file $O/traffic_c2.csv \
   python bench.py --steps 5 --warmup 3 --no-cpu-baseline --parity-full 0 > $O/ncu_traffic_c2.log 2>&1
python tools/ncu_traffic.py $O/traffic_c2.csv --steps 5 --wbm-per-step 1 --build $SHA --out $O/traffic_c2.json > /dev/null 2>&1 \
  && cp $O/traffic_c2.json profiles/traffic_c2.json
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum \
   --clock-control none -k regex:"k_|Device" --csv --log-file $O/traffic_c4.csv \
   python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline --parity-full 0 > $O/ncu_traffic_c4.log 2>&1
python tools/ncu_traffic.py $O/traffic_c4.csv --steps 3 --wbm-per-step 1 --build $SHA --out $O/traffic_c4.json > /dev/null 2>&1 \
  && cp $O/traffic_c4.json profiles/traffic_c4.json
rm -f $O/traffic_c2.csv $O/traffic_c4.csv
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.log
timeout 900 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > $O/c4.json 2> $O/c4.log
timeout 900 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu-baseline --parity-full 0 > $O/c3.json 2> $O/c3.log
tail -2 $O/pytest_gpu.log; tail -1 $O/smoke.log
for c in bench c4 c3; do python tools/bench_brief.py $O/$c.json $c; done

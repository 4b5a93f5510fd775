#!/usr/bin/env bash
# Round 2, call W: k_merge_refresh with the batch keys held in lanes (ballots instead of a search per moved
# element) — parity tests on the default build, then C4 / C2 across library variants (register budget 4/5/6
# CTAs per SM, and the per-element search).
O=gpurun_out/w; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stream.py tests/test_gpu_scale.py tests/test_gpu_group.py -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
tail -3 $O/pytest.log
for r in 1 2; do for v in b200 nokl mw6 mw4; do
  BDSM_LIB=$PWD/paper_2401_17018_b200/libbdsm_$v.so timeout 900 python tools/ab_env.py --config C4 --steps 4 --warmup 3 --rounds 1 --variant $v: > $O/c4_${v}_$r.txt 2> $O/c4_${v}_$r.log
  tail -1 $O/c4_${v}_$r.txt
done; done
for v in b200 nokl mw6; do
  BDSM_LIB=$PWD/paper_2401_17018_b200/libbdsm_$v.so timeout 900 python tools/ab_env.py --config C2 --steps 10 --warmup 3 --rounds 3 --variant $v: > $O/c2_$v.txt 2> $O/c2_$v.log
  tail -1 $O/c2_$v.txt
done

#!/usr/bin/env bash
# Round 2, call Y: every BASELINE config with the final build (C1, C3, C5 clique, C5 cycle; C2 and C4 are in call X),
# plus the parity-at-scale check of C3 / C4 prefixes.
O=gpurun_out/y; mkdir -p $O
timeout 900 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu-baseline --parity-full 0 > $O/c3.json 2> $O/c3.log
timeout 600 python bench.py --config C1 --steps 5 --warmup 3 --no-cpu-baseline > $O/c1.json 2> $O/c1.log
timeout 600 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline --coalesce > $O/c5.json 2> $O/c5.log
timeout 900 python bench.py --config C5cycle --steps 3 --warmup 3 --no-cpu-baseline --parity-full 0 --coalesce > $O/c5cyc.json 2> $O/c5cyc.log
for c in c3 c1 c5 c5cyc; do python tools/bench_brief.py $O/$c.json $c; done

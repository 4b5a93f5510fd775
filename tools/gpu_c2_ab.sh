#!/usr/bin/env bash
# Parity tests, then a 12-step C2 line (negative-phase ms per step for A/B against the previous build).
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for i in 1 2; do
timeout 600 python bench.py --steps 12 --warmup 3 --no-cpu-baseline ${BENCH_ARGS:-} 2>/dev/null | python -c "import json,sys; b=json.load(sys.stdin); print(round(b['value']), round(b['e2e']['value']), round(b['ms_per_step'],4), 'neg', [round(s['neg_ms'],3) for s in b['per_step']], 'pos', [round(s['pos_ms'],3) for s in b['per_step']])"
done

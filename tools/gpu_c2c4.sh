#!/usr/bin/env bash
# GPU parity tests, then C2 and C4 bench lines with the per-phase split.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.log
timeout 1800 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.log
python - <<'PY'
import json
for c in ("C2", "C4"):
    try:
        b = json.load(open(f"gpurun_out/bench_{c}.json"))
    except Exception as e:
        print(c, "failed", e); continue
    print(c, round(b["value"]), round(b["e2e"]["value"]), round(b["ms_per_step"], 3),
          [(round(s["ms"], 3), round(s["neg_ms"], 3), round(s["merge_ms"], 3), round(s["pos_ms"], 3)) for s in b["per_step"]][:3],
          b["counts"]["e2e_equals_device_path"])
PY

"""One-line summary of a bench.py JSON line: value, e2e, ms per step, per-kernel split if present."""
import json
import sys

try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    lat = d.get("latency") or {}
    print(sys.argv[2], "value", round(d["value"]), "e2e", round(d["e2e"]["value"]), "ms", round(d["ms_per_step"], 4),
          "merge_ms", [round(x, 3) for x in lat.get("merge_ms", [])], "parity", (d.get("parity_full") or {}).get("equal"))
except Exception as ex:  # noqa: BLE001
    print(sys.argv[2], "FAILED", ex)

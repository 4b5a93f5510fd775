#!/usr/bin/env python
"""Per-kernel DRAM / L2 traffic of the timed steps from an ncu metrics CSV.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum \
        --clock-control none --csv --log-file traffic.csv python bench.py --steps S --warmup W ...
    python tools/ncu_traffic.py traffic.csv --steps S --build <sha> [--out profiles/x.json]

Only this library's kernels (k_*) and CUB's are kept.  The launches of one
bench step are found from the per-step k_wbm count (one query: 2 per step one
batch at a time, 1 in the pipelined stream where the positive phase of batch i
and the negative phase of batch i+1 share a launch); the summary is per step of
the last S steps,
so bench.py can put physical bytes beside its live per-step kernel time.
"""
import argparse
import collections
import csv
import json
import re
import sys


def short(name):
    m = re.search(r"(k_\w+)", name)
    if m:
        return m.group(1)
    if "cub" in name.lower() or "Device" in name:
        m = re.search(r"(Device\w+Kernel\w*)", name)
        return "cub::" + (m.group(1) if m else "kernel")
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--steps", type=int, required=True)
    ap.add_argument("--wbm-per-step", type=int, default=2)
    ap.add_argument("--build", default=None)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    rows = []
    with open(args.csv) as f:
        lines = [l for l in f if l.startswith('"')]
    rd = csv.DictReader(lines)
    launches = collections.OrderedDict()
    for r in rd:
        k = short(r["Kernel Name"])
        if k is None:
            continue
        lid = int(r["ID"])
        d = launches.setdefault(lid, {"kernel": k})
        v = r["Metric Value"].replace(",", "")
        try:
            d[r["Metric Name"]] = float(v)
        except ValueError:
            pass
    seq = list(launches.values())
    wbm_idx = [i for i, d in enumerate(seq) if d["kernel"] == "k_wbm"]
    need = args.steps * args.wbm_per_step
    if len(wbm_idx) < need:
        sys.exit(f"only {len(wbm_idx)} k_wbm launches, need {need}")
    # the timed steps: every launch after the k_wbm that closes the step before them
    prev_end = wbm_idx[-need - 1] if len(wbm_idx) > need else -1
    timed = seq[prev_end + 1:]
    per = collections.defaultdict(lambda: collections.Counter())
    for d in timed:
        c = per[d["kernel"]]
        c["launches"] += 1
        c["ns"] += d.get("gpu__time_duration.sum", 0)
        c["dram_read"] += d.get("dram__bytes_read.sum", 0)
        c["dram_write"] += d.get("dram__bytes_write.sum", 0)
        c["l2_bytes"] += d.get("lts__t_bytes.sum", 0)
    S = args.steps
    out = {"source": args.csv, "build": args.build, "steps": S,
           "note": "ncu --clock-control none, metrics pass (cold cache, serialised launches); per step = sum over "
                   "the step's launches / steps",
           "kernels": {}}
    tot_ns = sum(c["ns"] for c in per.values())
    for k, c in sorted(per.items(), key=lambda kv: -kv[1]["ns"]):
        out["kernels"][k] = {
            "launches_per_step": c["launches"] / S,
            "ms_per_step": c["ns"] / S / 1e6,
            "share_of_step": c["ns"] / tot_ns if tot_ns else 0,
            "dram_bytes_per_step": (c["dram_read"] + c["dram_write"]) / S,
            "dram_read_per_step": c["dram_read"] / S,
            "dram_write_per_step": c["dram_write"] / S,
            "l2_bytes_per_step": c["l2_bytes"] / S,
            "dram_GBps": (c["dram_read"] + c["dram_write"]) / c["ns"] if c["ns"] else 0,
            "l2_GBps": c["l2_bytes"] / c["ns"] if c["ns"] else 0,
        }
    s = json.dumps(out, indent=1)
    print(s)
    if args.out:
        with open(args.out, "w") as f:
            f.write(s + "\n")


if __name__ == "__main__":
    main()

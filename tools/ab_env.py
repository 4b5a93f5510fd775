"""A/B of engine tuning knobs (BDSM_TUNE_* environment variables) on one workload.

    python tools/ab_env.py --config C4 --steps 4 --warmup 3 --rounds 2 \
        --variant base: --variant g16:BDSM_TUNE_SMALL_GROUP=16 ...

The workload is generated once; every variant builds its own engine (the
knobs are read when an engine is created), streams the warm-up batches, then
times the rest as one pipelined stream from HBM (bench.py's `value`).  The
variants alternate over `--rounds`, and every variant's counts must equal the
first one's.  Prints one JSON line per (round, variant) and a summary.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workload as W  # noqa: E402


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--rounds", type=int, default=2)
    ap.add_argument("--coalesce", action="store_true")
    ap.add_argument("--variant", action="append", required=True, help="name:VAR=val,VAR=val")
    args = ap.parse_args()
    import paper_2401_17018_b200 as bd

    dev = torch.device("cuda", 0)
    nb = args.warmup + args.steps
    t0 = time.time()
    wl = W.build(args.config, nb, device=dev, batch=args.batch)
    print(f"workload {args.config} {wl.meta} gen {time.time() - t0:.1f}s", file=sys.stderr, flush=True)
    dev_batches = [torch.from_numpy(b.view(np.uint32).reshape(-1, 4).copy()).to(dev) for b in wl.batches]
    variants = []
    for v in args.variant:
        name, _, kv = v.partition(":")
        env = dict(x.split("=", 1) for x in kv.split(",") if x)
        variants.append((name, env))
    base_counts = None
    res = {name: [] for name, _ in variants}
    for rnd in range(args.rounds):
        for name, env in variants:
            saved = {k: os.environ.get(k) for k in env}
            os.environ.update(env)
            try:
                t1 = time.time()
                e = bd.Engine(wl.labels, wl.src, wl.dst, device=0, coalesce=args.coalesce)
                e.add_query(wl.qlabels, wl.qedges)
                build_s = time.time() - t1
                warm = e.match_stream_device([dev_batches[i].data_ptr() for i in range(args.warmup)],
                                             [len(wl.batches[i]) for i in range(args.warmup)])
                torch.cuda.synchronize()
                rs = e.match_stream_device([dev_batches[i].data_ptr() for i in range(args.warmup, nb)],
                                           [len(wl.batches[i]) for i in range(args.warmup, nb)])
                counts = [(r.positive[0], r.negative[0]) for r in list(warm) + list(rs)]
                ms = sum(r.stats["ms_device"] for r in rs) / len(rs)
                merge = [round(r.stats.get("ms_merge_kernel", 0), 3) for r in rs]
                e.close()
            finally:
                for k, old in saved.items():
                    if old is None:
                        os.environ.pop(k, None)
                    else:
                        os.environ[k] = old
            if base_counts is None:
                base_counts = counts
            ups = wl.meta["batch"] * 1e3 / ms
            res[name].append(ups)
            print(json.dumps({"round": rnd, "variant": name, "env": env, "ms_per_batch": ms, "updates_per_s": ups,
                              "ms_merge": merge, "counts_equal_first": counts == base_counts,
                              "engine_build_s": round(build_s, 1)}), flush=True)
            if counts != base_counts:
                print(f"COUNT MISMATCH in {name}", file=sys.stderr, flush=True)
                return 1
    for name, _ in variants:
        print(f"{name:>12}: " + " ".join(f"{x / 1e6:.2f}M" for x in res[name]) +
              f"  median {statistics.median(res[name]) / 1e6:.2f}M", flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())

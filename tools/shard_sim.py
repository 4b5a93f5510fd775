#!/usr/bin/env python
"""Multi-GPU prediction from one GPU.

    python tools/shard_sim.py --config C4 --worlds 1,2,4,8 [--steps 3 --warmup 3] [--out FILE]

For every world size W and rank r < W, an engine with shard (r, W) replays the
same stream on the one visible GPU — the graph replicated, every rank applying
the whole batch, counting only its share of the work units — and each step's
device time is recorded.  The predicted W-GPU step is the slowest rank's step
plus the two collectives of a real run (NCCL broadcast of the batch and a
16-byte all-reduce per query, at the measured NVLink peer bandwidth plus a
fixed latency).  The per-rank counts must sum to the 1-rank counts batch by
batch.  Prints one JSON object.
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

import paper_2401_17018_b200 as bd  # noqa: E402
import workload as W  # noqa: E402

NVLINK_GBPS = 770.0      # measured peer copy per direction (B200_PROFILING.md)
COLL_LATENCY_MS = 0.015  # per collective, small-message NCCL latency on NVSwitch (estimate)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--worlds", default="1,2,4,8")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--out", default=None)
    ap.add_argument("--no-stream", dest="stream", action="store_false",
                    help="one apply per batch instead of the pipelined stream")
    args = ap.parse_args()
    worlds = [int(w) for w in args.worlds.split(",")]
    dev = torch.device("cuda", 0)
    nb = args.warmup + args.steps
    t0 = time.time()
    wl = W.build(args.config, nb, device=dev, batch=args.batch)
    gen_s = time.time() - t0
    dev_batches = [torch.from_numpy(b.view(np.uint32).reshape(-1, 4).copy()).to(dev) for b in wl.batches]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    bcast_ms = 16 * wl.meta["batch"] / (NVLINK_GBPS * 1e9) * 1e3 + COLL_LATENCY_MS
    reduce_ms = COLL_LATENCY_MS
    res = {"config": args.config, "V": wl.meta["V"], "E": wl.meta["E"], "batch": wl.meta["batch"],
           "mode": "pipelined stream per rank" if args.stream else "one apply per batch per rank",
           "steps": args.steps, "warmup": args.warmup, "gen_s": gen_s,
           "collectives_ms": {"broadcast": bcast_ms, "allreduce": reduce_ms,
                              "model": f"16 B/update at {NVLINK_GBPS} GB/s + {COLL_LATENCY_MS} ms per collective"},
           "worlds": {}}
    base_counts = None
    for Wd in worlds:
        ranks = []
        counts_sum = None
        for r in range(Wd):
            eng = bd.Engine(wl.labels, wl.src, wl.dst, device=0, shard_rank=r, shard_world=Wd)
            eng.add_query(wl.qlabels, wl.qedges)
            per, cnt = [], []
            if args.stream:  # warm-up and timed batches each as one pipelined stream
                for lo, hi, keep in ((0, args.warmup, False), (args.warmup, nb, True)):
                    flush.zero_()
                    torch.cuda.synchronize()
                    rs = eng.match_stream_device([dev_batches[i].data_ptr() for i in range(lo, hi)],
                                                 [len(wl.batches[i]) for i in range(lo, hi)])
                    for rr in rs:
                        cnt.append((rr.positive[0], rr.negative[0]))
                        if keep:
                            s = rr.stats
                            per.append({k: s[k] for k in ("ms_device", "ms_match_kernel", "ms_merge_kernel",
                                                          "work_items")})
            for i in range(nb) if not args.stream else []:
                flush.zero_()
                torch.cuda.synchronize()
                rr = eng.match_batch_device(dev_batches[i].data_ptr(), len(wl.batches[i]))
                cnt.append((rr.positive[0], rr.negative[0]))
                if i >= args.warmup:
                    s = rr.stats
                    per.append({k: s[k] for k in ("ms_device", "ms_negative", "ms_update", "ms_positive",
                                                  "ms_match_kernel", "ms_merge_kernel", "work_items")})
            eng.close()
            torch.cuda.empty_cache()
            counts_sum = cnt if counts_sum is None else [(a[0] + b[0], a[1] + b[1]) for a, b in zip(counts_sum, cnt)]
            ranks.append(per)
        if base_counts is None:
            base_counts = counts_sum
        # the stream's per-batch times are pipeline steps: compare the ranks'
        # total time over the timed batches
        if args.stream:
            tot = [sum(p["ms_device"] for p in ranks[r]) for r in range(Wd)]
            step_max = [max(tot) / args.steps] * args.steps
        else:
            step_max = [max(ranks[r][k]["ms_device"] for r in range(Wd)) for k in range(args.steps)]
        kmax = [max(ranks[r][k]["ms_match_kernel"] for r in range(Wd)) for k in range(args.steps)]
        repl = [statistics.mean(ranks[r][k]["ms_device"] - ranks[r][k]["ms_match_kernel"] for r in range(Wd))
                for k in range(args.steps)]
        # one broadcast of the batch and one count reduction per step (a stream
        # needs only one reduction at its end; counted per step to stay safe)
        pred = [s + (bcast_ms + reduce_ms if Wd > 1 else 0.0) for s in step_max]
        res["worlds"][str(Wd)] = {
            "predicted_ms_per_step": statistics.mean(pred),
            "max_rank_step_ms": statistics.mean(step_max),
            "max_rank_match_kernel_ms": statistics.mean(kmax),
            "replicated_ms_mean": statistics.mean(repl),
            "per_rank_step_ms": [statistics.mean(p["ms_device"] for p in ranks[r]) for r in range(Wd)],
            "per_rank_match_kernel_ms": [statistics.mean(p["ms_match_kernel"] for p in ranks[r]) for r in range(Wd)],
            "counts_sum_equal_1rank": counts_sum == base_counts,
        }
        print(f"[shard_sim] {args.config} W={Wd}: {res['worlds'][str(Wd)]['predicted_ms_per_step']:.3f} ms/step",
              file=sys.stderr, flush=True)
    w1 = res["worlds"].get("1", {}).get("predicted_ms_per_step")
    for k, v in res["worlds"].items():
        v["predicted_speedup"] = w1 / v["predicted_ms_per_step"] if w1 else None
        v["predicted_updates_per_s"] = wl.meta["batch"] / (v["predicted_ms_per_step"] / 1e3)
    s = json.dumps(res)
    print(s, flush=True)
    if args.out:
        with open(args.out, "w") as f:
            f.write(s + "\n")
    return 0


if __name__ == "__main__":
    sys.exit(main())

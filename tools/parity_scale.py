#!/usr/bin/env python
"""Parity at scale (TEST INFRASTRUCTURE, run on the GPU box).

    python tools/parity_scale.py --config C3 --batches 3 --prefix 100 [--batch N] [--out FILE]

Generates a BASELINE config's workload on the GPU, replays it through the CUDA
engine (C ABI) and through the CPU restatement (oracle/oracle_bench, pinned to
the reference on tests/golden/ by counts and MatchStats) with the same
sub-batch protocol — the first P updates of each batch counted, the rest
applied (P = 0: whole batches) — and compares positive/negative counts and the
reference's dfs_visits batch by batch (SURVEY.md §8(c) "Parity at scale").
Prints one JSON object.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import torch  # noqa: E402

import paper_2401_17018_b200 as bd  # noqa: E402
import workload as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--batches", type=int, default=3)
    ap.add_argument("--prefix", type=int, default=0)
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--timeout", type=float, default=1800)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()

    t0 = time.time()
    wl = W.build(args.config, args.batches, device="cuda", batch=args.batch)
    gen_s = time.time() - t0
    eng = bd.Engine(wl.labels, wl.src, wl.dst, device=0)
    eng.add_query(wl.qlabels, wl.qedges)
    ours, visits, ms = [], [], []
    for b in wl.batches:
        P = args.prefix if args.prefix and args.prefix < len(b) else len(b)
        r = eng.match_batch(b[:P])
        ours.append((r.positive[0], r.negative[0]))
        visits.append(r.stats["dfs_visits"])
        ms.append(r.stats["ms_device"])
        if P < len(b):
            eng.match_batch(b[P:])
    eng.close()
    torch.cuda.empty_cache()

    tmp = tempfile.mkdtemp(prefix="bdsm_parity_")
    path = os.path.join(tmp, "workload.bin")
    W.write_file(wl, path)
    meta = wl.meta
    del wl
    exe = os.path.join(REPO, "oracle", "oracle_bench")
    cmd = [exe, path, "--threads", str(os.cpu_count() or 1), "--batches", str(args.batches)]
    if args.prefix:
        cmd += ["--prefix", str(args.prefix)]
    t1 = time.time()
    try:
        out = subprocess.run(cmd, capture_output=True, text=True, timeout=args.timeout).stdout
    except subprocess.TimeoutExpired as e:
        out = e.stdout.decode() if isinstance(e.stdout, bytes) else (e.stdout or "")
    cpu_s = time.time() - t1
    os.unlink(path)
    os.rmdir(tmp)
    lines = [json.loads(l) for l in out.splitlines() if l.startswith("{")]
    per = [l for l in lines if "batch" in l]
    summ = [l for l in lines if l.get("summary")]
    ref = [(l["positive"], l["negative"]) for l in per]
    ref_v = [l["dfs_visits_pruned"] for l in per]
    ref_tree = [l["dfs_visits"] for l in per]
    res = {
        "config": args.config, "V": meta["V"], "E": meta["E"], "d_max": meta["d_max"], "batch": meta["batch"],
        "prefix": args.prefix or meta["batch"], "batches_checked": len(per), "batches": args.batches,
        "ours": ours, "restatement": ref, "counts_equal": ours[:len(ref)] == ref and len(ref) == args.batches,
        "dfs_visits_ours": visits, "dfs_visits_restatement": ref_v, "dfs_visits_reference_tree": ref_tree,
        "dfs_visits_equal": visits[:len(ref_v)] == ref_v,
        "max_count": max([max(p) for p in ref] or [0]), "ge_2_32": any(max(p) >= 2 ** 32 for p in ref),
        "gpu_ms_per_subbatch": ms, "cpu_s": cpu_s, "gen_s": gen_s,
        "cpu_summary": summ[0] if summ else None, "cores": os.cpu_count(),
    }
    s = json.dumps(res)
    print(s, flush=True)
    if args.out:
        with open(args.out, "w") as f:
            f.write(s + "\n")
    return 0 if res["counts_equal"] else 1


if __name__ == "__main__":
    sys.exit(main())

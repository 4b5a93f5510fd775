#!/usr/bin/env python
"""Diagnostics of the C2 workload on one GPU: plan (orders, independent tails)
and, with a -DBDSM_TRACE build (BDSM_LIB=...), per-phase item traces.

  BDSM_LIB=path/to/trace.so python tools/diag_c2.py [--batches N] [--config C2]
"""
import argparse
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2401_17018_b200 as bd  # noqa: E402
import workload as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--batches", type=int, default=6)
    ap.add_argument("--chunk", type=int, default=64)
    ap.add_argument("--quiet", action="store_true")
    args = ap.parse_args()
    wl = W.build(args.config, args.batches)
    e = bd.Engine(wl.labels, wl.src, wl.dst, device=0, chunk=args.chunk)
    q = e.add_query(wl.qlabels, wl.qedges)
    print("query", wl.qlabels, wl.qedges)
    for ei in range(len(wl.qedges)):
        print(f"  edge {ei} {wl.qedges[ei]}: order {e.order(q, ei)} tail {e.tail(q, ei)}")
    print("columns", e.column_sizes(q))
    for bi, b in enumerate(wl.batches):
        r = e.match_batch(b)
        st = r.stats
        tr = e.debug_trace()
        print(f"batch {bi}: +{r.positive[0]} -{r.negative[0]} ms neg {st['ms_negative']:.3f} "
              f"upd {st['ms_update']:.3f} pos {st['ms_positive']:.3f} visits {st['dfs_visits']} "
              f"kbytes {st['bytes_kernel']/1e9:.2f}G refbytes {st['bytes_phase']/1e9:.2f}G")
        for ph, t in ([] if args.quiet else tr.items()):
            if t["t_last"] and t["t_first"] != 2**64 - 1:
                span = (t["t_last"] - t["t_first"]) / 1e6
                print(f"   {ph}: span {span:.3f} ms busy {t['busy_ns']/1e6:.1f} warp-ms "
                      f"max item {t['max_item_ns']/1e6:.3f} ms (kind {t['max_item'] >> 8} level {t['max_item'] & 255}) "
                      f"static {t['static_items']} donated {t['donated_items']}")
                dg = t["mx_anchor_deg"]
                print(f"      longest item: chunks {t['mx_chunks']} tail chunks {t['mx_tail_chunks']} "
                      f"big leaf misses {t['mx_big_leaf']} donations {t['mx_donations']} anchor deg {dg >> 32}/{dg & 0xffffffff} "
                      f"us: donate {t['mx_cy_donate']/1965:.0f} filter {t['mx_cy_filter']/1965:.0f} "
                      f"leaf {t['mx_cy_leaf']/1965:.0f} setup {t['mx_cy_setup']/1965:.0f}")
                print(f"      chunks/level {t['chunks'][:len(wl.qlabels)]} setups/level {t['setups'][:len(wl.qlabels)]}")


if __name__ == "__main__":
    main()

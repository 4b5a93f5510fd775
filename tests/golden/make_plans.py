#!/usr/bin/env python
"""Regenerates tests/golden/plans.json from the UNMODIFIED reference
(oracle/_ref/libbdsm_refshim.so, built from /root/reference by `make -C oracle
ref`): for the golden instances' initial graphs, the reference's matching
order of every query edge (generate_matching_order, src/query_analysis.cpp
:358-363, over its CandidateTable) and the candidate column sizes it used.
tests/test_planner.py checks the B200 host planner against it on CPU."""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, ".."))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))

import golden_util as gu  # noqa: E402
from oracle_py import ref_plan_orders  # noqa: E402


def main():
    out = []
    for suite in ("fig1", "skewed", "matcher_random", "edge_labeled", "acceptance_random", "streams"):
        for inst in gu.load(suite):
            vl, eu, ev, el, ql, qe, _ = gu.instance_arrays(inst)
            try:
                orders, cols = ref_plan_orders(vl, eu, ev, el, ql, qe)
            except Exception as ex:  # disconnected / invalid queries are the error tests' business
                print("skip", suite, inst["name"], ex)
                continue
            out.append({"suite": suite, "name": inst["name"], "qlabels": ql,
                        "qedges": [[a, b, -1 if c is None else c] for a, b, c in qe],
                        "column_sizes": cols, "orders": orders})
    with open(os.path.join(HERE, "plans.json"), "w") as f:
        json.dump(out, f)
    print(len(out), "plans")


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Golden instances through the engine, for compute-sanitizer (no torch import).

    compute-sanitizer --tool memcheck  python tools/sanitize_golden.py [suite ...]
    compute-sanitizer --tool racecheck python tools/sanitize_golden.py fig1 skewed

Runs every batch of the chosen golden suites one batch at a time and as a
pipelined stream, and checks the counts against the reference's (the
sanitizer reports memory errors / shared-memory races of the kernels).
Prints one line per suite and exits non-zero on a count mismatch.
"""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))

import golden_util as gu  # noqa: E402
import paper_2401_17018_b200 as bd  # noqa: E402


def main():
    suites = sys.argv[1:] or ["fig1", "skewed", "matcher_random", "edge_labeled", "streams"]
    bad = 0
    for suite in suites:
        n_inst = n_batch = 0
        for inst in gu.load(suite):
            vl, eu, ev, el, ql, qe, batches = gu.instance_arrays(inst)
            for mode in ("single", "stream"):
                e = bd.Engine(vl, eu, ev, el, chunk=8)
                e.add_query(ql, qe)
                nonempty = [(b, x) for b, x in zip(batches, inst["expect"]) if len(b)]
                if mode == "single":
                    got = [e.match_batch(b) for b, _ in nonempty]
                else:
                    got = e.match_stream([b for b, _ in nonempty]) if nonempty else []
                for r, (_, x) in zip(got, nonempty):
                    n_batch += 1
                    if (r.positive[0], r.negative[0]) != (x["pos"], x["neg"]):
                        bad += 1
                        print("MISMATCH", suite, inst["name"], mode, flush=True)
                e.close()
            n_inst += 1
        print(f"{suite}: {n_inst} instances, {n_batch} batches checked", flush=True)
    print("mismatches", bad)
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())

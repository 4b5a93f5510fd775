#!/usr/bin/env python
"""Regenerates tests/golden/cli/ from the UNMODIFIED reference's `bdsm run`
path (oracle/_ref/ref_cli: load/generate -> run_pipeline with coalesce off ->
emit_report), run in the build container (needs /root/reference to build it).

Each case directory holds the inputs (graph, query/stream files or generator
specs), what the reference wrote (query_<i>.txt, stream.txt, deltas.csv) and
its stdout summary line.  tests/test_cli.py checks the B200 CLI against them:
generators byte-identical on CPU, deltas/summary identical on the GPU.
"""
import json
import os
import random
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
OUT = os.path.join(HERE, "cli")
REF_CLI = os.path.join(REPO, "oracle", "_ref", "ref_cli")

FIG1_G = ["v 0 1", "v 1 1", "v 2 2", "v 3 2", "v 4 2", "v 5 2", "v 6 2", "v 7 4", "v 8 4", "v 9 4"]
# tests/support/fig1.hpp:29-37 (the running example's 13 edges)
FIG1_E = [(0, 3), (0, 4), (0, 6), (1, 5), (1, 6), (2, 3), (2, 4), (2, 7), (3, 8), (4, 5), (4, 8), (5, 6), (5, 9)]
FIG1_Q = ["v 0 1", "v 1 2", "v 2 2", "v 3 4", "e 0 1", "e 0 2", "e 1 2", "e 1 3"]


def write(path, lines):
    with open(path, "w") as f:
        f.write("\n".join(lines) + "\n")


def random_graph(path, V, E, L, seed, elabels=0):
    rng = random.Random(seed)
    lines = [f"v {v} {rng.randrange(L)}" for v in range(V)]
    pairs = set()
    # power-law-ish: half the endpoints from a small hub set
    hubs = list(range(max(2, V // 20)))
    while len(pairs) < E:
        a = rng.choice(hubs) if rng.random() < 0.3 else rng.randrange(V)
        b = rng.randrange(V)
        if a != b:
            pairs.add((min(a, b), max(a, b)))
    for a, b in sorted(pairs):
        lines.append(f"e {a} {b}" + (f" {rng.randrange(elabels)}" if elabels else ""))
    write(path, lines)


def run_case(name, graph, qspec, sspec, seed, dump=True):
    d = os.path.join(OUT, name)
    ref_out = os.path.join(d, "ref")
    shutil.rmtree(ref_out, ignore_errors=True)
    r = subprocess.run([REF_CLI, graph, qspec, sspec, str(seed), ref_out] + (["dump"] if dump else []),
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    meta = {"qspec": qspec, "sspec": sspec, "seed": seed, "summary": r.stdout.strip(), "dump_matches": dump}
    for f in ("latency.csv", "stages.csv", "utilization.csv"):
        os.remove(os.path.join(ref_out, f))  # timing-dependent, headers are checked in tests
    with open(os.path.join(d, "case.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print(name, meta["summary"])


def main():
    subprocess.run(["make", "-s", "-C", os.path.join(REPO, "oracle"), "ref"], check=True)
    shutil.rmtree(OUT, ignore_errors=True)
    os.makedirs(OUT)
    # Fig. 1 (SURVEY.md §8(c) CLI golden): one batch, then the same updates as three batches
    d = os.path.join(OUT, "fig1")
    os.makedirs(d)
    write(os.path.join(d, "g.txt"), FIG1_G + [f"e {a} {b}" for a, b in FIG1_E])
    write(os.path.join(d, "q.txt"), FIG1_Q)
    write(os.path.join(d, "s1.txt"), ["+ 0 2", "+ 1 4", "- 4 5"])
    write(os.path.join(d, "s3.txt"), ["+ 0 2", "", "+ 1 4", "", "- 4 5"])
    for s in ("s1", "s3"):
        os.makedirs(os.path.join(OUT, f"fig1_{s}"))
        run_case(f"fig1_{s}", os.path.join(d, "g.txt"), "q:" + os.path.join(d, "q.txt"),
                 "s:" + os.path.join(d, s + ".txt"), 1)
    # generated workloads through the reference's own generators
    cases = [
        ("gen_sparse_mixed", 400, 2400, 3, 0, "g:sparse,5,3", "s:0.05,mixed,4", 5, True),
        ("gen_tree_insert", 300, 1500, 2, 0, "g:tree,4,2", "s:0.08,insert,3", 11, False),
        ("gen_dense_delete", 200, 1800, 2, 0, "g:dense,4,2", "s:0.05,delete,2", 3, True),
        ("gen_kcore_mixed", 300, 2000, 3, 0, "g:sparse,4,2", "s:0.05,mixed,3,4", 21, True),
        ("gen_elabel_mixed", 250, 1500, 2, 2, "g:sparse,4,2", "s:0.06,mixed,3", 8, True),
        # the paper's 50-query sets: more queries than one 32-bit mask
        ("gen_sparse50_mixed", 1500, 9000, 2, 0, "g:sparse,6,50", "s:0.02,mixed,3", 13, False),
    ]
    for name, V, E, L, EL, q, s, seed, dump in cases:
        d = os.path.join(OUT, name)
        os.makedirs(d)
        random_graph(os.path.join(d, "g.txt"), V, E, L, seed, EL)
        run_case(name, os.path.join(d, "g.txt"), q, s, seed, dump)
    # relative paths in case.json
    for name in os.listdir(OUT):
        p = os.path.join(OUT, name, "case.json")
        if os.path.exists(p):
            with open(p) as f:
                m = json.load(f)
            for k in ("qspec", "sspec"):
                m[k] = m[k].replace(OUT + "/", "")
            m["summary"] = m["summary"].replace(os.path.join(OUT, name, "ref") + "/", "OUT/")
            with open(p, "w") as f:
                json.dump(m, f, indent=1)


if __name__ == "__main__":
    sys.exit(main())

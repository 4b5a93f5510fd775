"""Loads the committed golden fixtures (tests/golden/*.json, generated from the
UNMODIFIED reference by tests/golden/make_golden.sh)."""
import json
import os

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
SUITES = ["fig1", "skewed", "matcher_random", "edge_labeled", "acceptance_random", "streams"]


def load(suite):
    with open(os.path.join(GOLDEN, suite + ".json")) as f:
        return json.load(f)


def instance_arrays(inst):
    """-> vlabels, eu, ev, elab(or None), qlabels, qedges, batches"""
    edges = inst["edges"]
    eu = [e[0] for e in edges]
    ev = [e[1] for e in edges]
    has = any(e[2] >= 0 for e in edges) or any(u[3] >= 0 for b in inst["batches"] for u in b)
    elab = [e[2] if e[2] >= 0 else 0xFFFFFFFF for e in edges] if has else None
    qedges = [(e[0], e[1], None if e[2] < 0 else e[2]) for e in inst["qedges"]]
    batches = [[(u[0], u[1], u[2], None if u[3] < 0 else u[3]) for u in b] for b in inst["batches"]]
    return inst["vlabels"], eu, ev, elab, inst["qlabels"], qedges, batches

"""Runs one golden instance through the engine (debug helper for the GPU box)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import golden_util as gu
import paper_2401_17018_b200 as bd

suite, idx = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0
inst = gu.load(suite)[idx]
vl, eu, ev, el, ql, qe, batches = gu.instance_arrays(inst)
e = bd.Engine(vl, eu, ev, el)
e.add_query(ql, qe)
for b, exp in zip(batches, inst["expect"]):
    r = e.match_batch(b)
    print(inst["name"], r.positive, r.negative, "expect", exp["pos"], exp["neg"], r.stats["dfs_visits"], exp["visits"])

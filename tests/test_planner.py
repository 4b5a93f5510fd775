"""The host planner (north_star item 2) against the reference's own plans
(tests/golden/plans.json, from the unmodified reference by
tests/golden/make_plans.py): given the reference's candidate column sizes,
bdsm_plan_order returns the reference's matching order for every query edge
(generate_matching_order -> try_order, src/query_analysis.cpp:295-363) —
including its tie-breaks.  (build_query_plan also re-orders the edges of
k-degenerated coalescing groups, :375-435; that only feeds the coalesced
search, out of scope per SURVEY F1.)  Pure host code: runs without a GPU.
Also checks the counted-tail classification on hand-made queries."""
import ctypes as C
import json
import os

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PLANS = os.path.join(REPO, "tests", "golden", "plans.json")


class _QueryDesc(C.Structure):
    _fields_ = [("num_vertices", C.c_uint32), ("vertex_labels", C.c_void_p), ("num_edges", C.c_uint32),
                ("a", C.c_void_p), ("b", C.c_void_p), ("edge_labels", C.c_void_p)]


def _lib():
    L = C.CDLL(os.path.join(REPO, "paper_2401_17018_b200", "libbdsm_b200.so"))
    L.bdsm_plan_order.restype = C.c_int
    L.bdsm_plan_order.argtypes = [C.POINTER(_QueryDesc), C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p]
    return L


def plan(L, qlabels, qedges, cols, edge):
    ql = np.asarray(qlabels, np.uint32)
    qa = np.asarray([e[0] for e in qedges], np.uint32)
    qb = np.asarray([e[1] for e in qedges], np.uint32)
    labelled = any(len(e) > 2 and e[2] is not None and e[2] >= 0 for e in qedges)
    qe = np.asarray([e[2] if len(e) > 2 and e[2] is not None and e[2] >= 0 else 0xFFFFFFFF for e in qedges],
                    np.uint32)
    d = _QueryDesc(len(ql), ql.ctypes.data, len(qa), qa.ctypes.data, qb.ctypes.data,
                   qe.ctypes.data if labelled else None)
    cs = np.asarray(cols, np.uint64)
    out = np.zeros(32, np.uint32)
    tail = np.zeros(1, np.uint32)
    n = L.bdsm_plan_order(C.byref(d), cs.ctypes.data, edge, out.ctypes.data, tail.ctypes.data)
    assert n >= 0, n
    return out[:n].tolist(), int(tail[0])


def test_orders_equal_reference():
    L = _lib()
    with open(PLANS) as f:
        plans = json.load(f)
    assert len(plans) > 500
    for p in plans:
        for e, ref_order in enumerate(p["orders"]):
            got, _ = plan(L, p["qlabels"], p["qedges"], p["column_sizes"], e)
            assert got == ref_order, (p["suite"], p["name"], e)


@pytest.mark.parametrize("labels,edges,cols,edge,tail", [
    # triangle + two pendant vertices (the C2 query shape): the leaves are counted
    ([4, 4, 13, 10, 1, 14], [(0, 1), (0, 3), (2, 3), (2, 4), (2, 5), (3, 4)], [120, 182, 87, 87, 120, 182], 1, 3),
    # 4-clique: no counted level beyond the last
    ([0, 0, 0, 0], [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)], [10, 10, 10, 10], 0, 3),
    # star with distinct leaf labels: everything after the anchor is counted
    ([0, 1, 2, 3], [(0, 1), (0, 2), (0, 3)], [5, 5, 5, 5], 0, 2),
    # star with equal leaf labels: injectivity couples the leaves, only the last is counted
    ([0, 1, 1, 1], [(0, 1), (0, 2), (0, 3)], [5, 5, 5, 5], 0, 3),
])
def test_counted_tail(labels, edges, cols, edge, tail):
    got_order, got_tail = plan(_lib(), labels, edges, cols, edge)
    assert sorted(got_order) == list(range(len(labels)))
    assert got_tail == tail, got_order


def test_disconnected_query_rejected():
    L = _lib()
    ql = np.asarray([0, 0, 0], np.uint32)
    qa, qb = np.asarray([0], np.uint32), np.asarray([1], np.uint32)
    d = _QueryDesc(3, ql.ctypes.data, 1, qa.ctypes.data, qb.ctypes.data, None)
    cs = np.ones(3, np.uint64)
    out = np.zeros(32, np.uint32)
    assert L.bdsm_plan_order(C.byref(d), cs.ctypes.data, 0, out.ctypes.data, None) == -2


def _orbits(labels, edges):
    import paper_2401_17018_b200 as bd
    return bd.plan_edge_orbits(labels, edges)


def test_edge_orbits_known_groups():
    """Exact coalescing plan: orbits of directed query edges under Aut(Q)."""
    k5 = [(i, j) for i in range(5) for j in range(i + 1, 5)]
    mult, n_aut = _orbits([0] * 5, k5)
    assert n_aut == 120 and sorted(m for m in mult if m) == [20]  # S5: one orbit of all 20
    c5 = [(i, (i + 1) % 5) for i in range(5)]
    mult, n_aut = _orbits([0] * 5, c5)
    assert n_aut == 10 and sorted(m for m in mult if m) == [10]   # D5
    # path a-b-c with equal labels: swapping a, c; orbits {(a,b),(c,b)}, {(b,a),(b,c)}
    mult, n_aut = _orbits([7, 7, 7], [(0, 1), (1, 2)])
    assert n_aut == 2 and mult == [2, 2, 0, 0]
    # labels break the symmetry: every directed edge searched once
    mult, n_aut = _orbits([1, 2, 3], [(0, 1), (1, 2)])
    assert n_aut == 1 and mult == [1, 1, 1, 1]
    # Fig. 1 query (labels A, B, B, C): u1/u2 are not interchangeable (u3 hangs on u1)
    mult, n_aut = _orbits([1, 2, 2, 4], [(0, 1), (0, 2), (1, 2), (1, 3)])
    assert n_aut == 1 and all(m == 1 for m in mult)
    # a triangle with one distinct label: swap of the two equal ones
    mult, n_aut = _orbits([1, 1, 2], [(0, 1), (1, 2), (0, 2)])
    assert n_aut == 2 and sum(mult) == 6 and max(mult) == 2


def test_edge_orbits_partition_every_direction():
    import random
    rng = random.Random(5)
    for _ in range(200):
        n = rng.randint(2, 7)
        edges = [(rng.randrange(i), i) for i in range(1, n)]
        extra = [(i, j) for i in range(n) for j in range(i + 1, n) if (i, j) not in edges and rng.random() < 0.3]
        edges += extra
        labels = [rng.randrange(2) for _ in range(n)]
        mult, n_aut = _orbits(labels, edges)
        assert sum(mult) == 2 * len(edges)
        assert n_aut >= 1

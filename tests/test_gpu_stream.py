"""The pipelined stream (bdsm_engine_apply_stream): the positive phase of batch
i and the negative phase of batch i+1 run as one launch of the matching
kernel.  Its results must equal one match_batch per batch — and therefore the
reference's — on every golden stream, with several queries, exact
coalescing, device-resident batches, a rejected batch in the middle, and the
work-item regrowth paths."""
import numpy as np
import pytest

import golden_util as gu
from oracle_py import Oracle

pytestmark = pytest.mark.gpu


def _engine(inst, **kw):
    import paper_2401_17018_b200 as bd
    vl, eu, ev, el, ql, qe, batches = gu.instance_arrays(inst)
    e = bd.Engine(vl, eu, ev, el, **kw)
    e.add_query(ql, qe)
    return e, batches


@pytest.mark.parametrize("suite", ["streams", "fig1", "skewed", "edge_labeled"])
def test_stream_equals_reference(suite):
    for inst in gu.load(suite):
        e, batches = _engine(inst)
        batches = [b for b in batches if len(b)]
        exp = [x for x, b in zip(inst["expect"], gu.instance_arrays(inst)[-1]) if len(b)]
        rs = e.match_stream(batches)
        assert len(rs) == len(batches)
        for bi, (r, x) in enumerate(zip(rs, exp)):
            assert (r.positive[0], r.negative[0]) == (x["pos"], x["neg"]), (inst["name"], bi)
        e.close()


def _random_workload(seed, V=600, E=9000, L=2, nb=6, bs=120):
    rng = np.random.default_rng(seed)
    pairs = set()
    while len(pairs) < E:
        a, b = (int(x) for x in rng.integers(0, V, 2))
        if a != b:
            pairs.add((min(a, b), max(a, b)))
    pairs = sorted(pairs)
    vl = rng.integers(0, L, V).astype(np.uint32)
    eu = np.array([p[0] for p in pairs], np.uint32)
    ev = np.array([p[1] for p in pairs], np.uint32)
    present = set(pairs)
    batches = []
    for _ in range(nb):
        batch, used = [], set()
        while len(batch) < bs:
            if rng.random() < 0.34:
                k = pairs[int(rng.integers(0, len(pairs)))]
                if k not in present or k in used:
                    continue
                batch.append((1, k[0], k[1]))
            else:
                a, b = (int(x) for x in rng.integers(0, V, 2))
                k = (min(a, b), max(a, b))
                if a == b or k in present or k in used:
                    continue
                batch.append((0, a, b))
            used.add((min(batch[-1][1], batch[-1][2]), max(batch[-1][1], batch[-1][2])))
        for op, a, b in batch:
            (present.add if op == 0 else present.discard)((min(a, b), max(a, b)))
        batches.append(batch)
    return vl, eu, ev, batches


QUERIES = [
    ([0, 1, 0, 1], [(0, 1), (1, 2), (2, 3), (3, 0)]),            # labelled 4-cycle
    ([0, 0, 1], [(0, 1), (1, 2), (0, 2)]),                       # triangle
    ([0, 1, 1, 0, 1], [(0, 1), (0, 2), (1, 2), (2, 3), (3, 4)]), # 5-vertex sparse
]


@pytest.mark.parametrize("coalesce", [False, True])
def test_stream_multi_query_equals_single_and_oracle(coalesce):
    import paper_2401_17018_b200 as bd
    vl, eu, ev, batches = _random_workload(3)
    es = bd.Engine(vl, eu, ev, coalesce=coalesce)
    e1 = bd.Engine(vl, eu, ev)
    o = Oracle(vl, eu, ev)
    for ql, qe in QUERIES:
        es.add_query(ql, qe)
        e1.add_query(ql, qe)
        o.add_query(ql, qe)
    rs = es.match_stream(batches)
    for bi, (b, r) in enumerate(zip(batches, rs)):
        r1 = e1.match_batch(b)
        pos, neg, st = o.apply_batch(b)
        assert (r.positive, r.negative) == (r1.positive, r1.negative) == (pos, neg), bi
        if not coalesce:
            assert r.stats["dfs_visits"] == r1.stats["dfs_visits"] == st[6], bi
    es.close()
    e1.close()


def test_stream_device_input():
    import torch
    import paper_2401_17018_b200 as bd
    vl, eu, ev, batches = _random_workload(5)
    e = bd.Engine(vl, eu, ev)
    o = Oracle(vl, eu, ev)
    for ql, qe in QUERIES[:2]:
        e.add_query(ql, qe)
        o.add_query(ql, qe)
    dev = [torch.from_numpy(bd.make_updates(b).view(np.uint32).reshape(-1, 4).copy()).cuda() for b in batches]
    rs = e.match_stream_device([t.data_ptr() for t in dev], [len(b) for b in batches])
    for b, r in zip(batches, rs):
        pos, neg, _ = o.apply_batch(b)
        assert (r.positive, r.negative) == (pos, neg)
    e.close()


@pytest.mark.parametrize("kind", ["missing_delete", "self_loop", "conflict"])
@pytest.mark.parametrize("at", [1, 2, 3])
def test_stream_rejected_batch_stops_there(kind, at):
    """A rejected batch (validation error found after the previous batch's
    merge, or a self-loop / conflicting pair found before it) stops the stream
    there: the batches before it are applied and reported, nothing of it."""
    import paper_2401_17018_b200 as bd
    vl, eu, ev, batches = _random_workload(7)
    present = {(int(a), int(b)) for a, b in zip(eu, ev)}
    for b in batches[:at]:
        for op, x, y in b:
            (present.add if op == 0 else present.discard)((min(x, y), max(x, y)))
    used = {(min(x, y), max(x, y)) for _, x, y in batches[at]}
    if kind == "missing_delete":  # found by the validation after the previous merge
        missing = next((a, b) for a in range(len(vl)) for b in range(a + 1, len(vl))
                       if (a, b) not in present and (a, b) not in used)
        bad = [(1, missing[0], missing[1])] + list(batches[at])
        err = bd.BatchError
    elif kind == "self_loop":  # found before the sort
        bad = list(batches[at]) + [(0, 5, 5)]
        err = ValueError
    else:  # the same pair twice: found after the sort
        bad = list(batches[at]) + [(batches[at][0][0], batches[at][0][2], batches[at][0][1])]
        err = ValueError
    stream = batches[:at] + [bad] + batches[at + 1:]
    e = bd.Engine(vl, eu, ev)
    o = Oracle(vl, eu, ev)
    for ql, qe in QUERIES:
        e.add_query(ql, qe)
        o.add_query(ql, qe)
    with pytest.raises(err) as ei:
        e.match_stream(stream)
    assert ei.value.done == at and len(ei.value.results) == at
    for b, r in zip(stream[:at], ei.value.results):
        pos, neg, _ = o.apply_batch(b)
        assert (r.positive, r.negative) == (pos, neg)
    if kind == "missing_delete":
        assert ei.value.failures and ei.value.failures[0][0] == 0
    # the engine holds exactly the batches before the bad one: the rest matches the oracle
    for b in batches[at:]:
        r = e.match_batch(b)
        pos, neg, _ = o.apply_batch(b)
        assert (r.positive, r.negative) == (pos, neg)
    e.close()


def test_stream_work_item_regrowth(monkeypatch):
    """A tiny initial work-item capacity forces negative- and positive-phase
    regrowth inside the stream (device abort chain, host rerun, resume)."""
    import paper_2401_17018_b200 as bd
    monkeypatch.setenv("BDSM_MAX_ITEMS", "16")
    vl, eu, ev, batches = _random_workload(9, nb=5, bs=200)
    e = bd.Engine(vl, eu, ev, chunk=8)
    o = Oracle(vl, eu, ev)
    for ql, qe in QUERIES:
        e.add_query(ql, qe)
        o.add_query(ql, qe)
    rs = e.match_stream(batches)
    assert any(r.stats["attempts"] > 1 or r.stats["reruns"] > 0 for r in rs)
    for b, r in zip(batches, rs):
        pos, neg, _ = o.apply_batch(b)
        assert (r.positive, r.negative) == (pos, neg)
    e.close()

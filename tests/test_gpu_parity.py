"""Parity of the CUDA engine (through the C ABI) against the reference's own
golden vectors: every batch of every golden instance must give exactly the
reference's |positive| / |negative| (bit-exact integer counts)."""
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


@pytest.mark.parametrize("suite", gu.SUITES)
def test_counts_equal_reference(suite):
    for inst in gu.load(suite):
        e, batches = _engine(inst)
        vl, eu, ev, el, ql, qe, _ = gu.instance_arrays(inst)
        o = Oracle(vl, eu, ev, el)
        o.add_query(ql, qe)
        for bi, (b, exp) in enumerate(zip(batches, inst["expect"])):
            r = e.match_batch(b)
            assert (r.positive[0], r.negative[0]) == (exp["pos"], exp["neg"]), (inst["name"], bi)
            # the engine applies dedupe_by_order when it generates candidates, so
            # its dfs_visits is the reference tree's minus the pruned subtrees:
            # exactly the restatement's pruned-visit count (pinned to the reference)
            _, _, st = o.apply_batch(b)
            assert st[0] == exp["visits"], (inst["name"], bi)
            assert r.stats["dfs_visits"] == st[6], (inst["name"], bi, r.stats["dfs_visits"], int(st[6]))
        e.close()


@pytest.mark.parametrize("chunk", [8, 16, 32, 96, 256])
def test_chunk_size_does_not_change_counts(chunk):
    for inst in gu.load("streams")[-4:] + gu.load("skewed"):
        e, batches = _engine(inst, chunk=chunk)
        for b, exp in zip(batches, inst["expect"]):
            r = e.match_batch(b)
            assert (r.positive[0], r.negative[0]) == (exp["pos"], exp["neg"]), inst["name"]


def test_fig1_singletons_and_graph_state():
    fig = {i["name"]: i for i in gu.load("fig1")}
    e, batches = _engine(fig["fig1_singletons"])
    got = [(r.positive[0], r.negative[0]) for r in (e.match_batch(b) for b in batches)]
    assert got == [(4, 0), (2, 0), (0, 2)]
    assert e.neighbors(0) == [2, 3, 4, 6]
    assert e.neighbors(4) == [0, 1, 2, 8]
    assert e.num_edges == 13 + 2 - 1


def test_batch_errors_all_or_nothing():
    import paper_2401_17018_b200 as bd
    fig = {i["name"]: i for i in gu.load("fig1")}
    e, _ = _engine(fig["fig1_batch"])
    with pytest.raises(bd.BatchError) as ei:
        e.match_batch([(0, 0, 2), (1, 0, 1), (0, 0, 3), (0, 0, 99)])
    assert ei.value.failures == [(1, 3), (2, 2), (3, 1)]
    assert "3 invalid update(s)" in str(ei.value)
    with pytest.raises(ValueError, match="self-loop update"):
        e.match_batch([(0, 0, 2), (0, 3, 3)])
    with pytest.raises(ValueError, match="conflicting updates on edge"):
        e.match_batch([(0, 1, 7), (1, 7, 1)])
    r = e.match_batch([(0, 0, 2), (0, 1, 4), (1, 4, 5)])  # nothing was applied before
    assert (r.positive, r.negative) == ([4], [0])


def test_pipelined_submit_wait():
    """bdsm_engine_submit_batch / bdsm_engine_wait (run_pipeline's stage
    overlap): the caller's buffer is free once submit returns, the counts equal
    match_batch's on every batch of a random stream, errors surface at wait
    with nothing applied, and one batch at most is in flight."""
    import numpy as np
    import paper_2401_17018_b200 as bd
    fig = {i["name"]: i for i in gu.load("fig1")}
    e, _ = _engine(fig["fig1_batch"])
    with pytest.raises(ValueError, match="no batch in flight"):
        e.wait()
    e.submit_batch([(0, 0, 2), (1, 0, 1), (0, 0, 3)])
    with pytest.raises(ValueError, match="already in flight"):
        e.submit_batch([(0, 1, 4)])
    with pytest.raises(bd.BatchError):
        e.wait()
    e.submit_batch([(0, 0, 2), (0, 3, 3)])
    with pytest.raises(ValueError, match="self-loop update"):
        e.wait()
    ups = bd.make_updates([(0, 0, 2), (0, 1, 4), (1, 4, 5)])
    e.submit_batch(ups)
    ups[:] = bd.make_updates([(1, 0, 3), (1, 0, 4), (1, 0, 6)])  # reused at once
    r = e.wait()
    assert (r.positive, r.negative) == ([4], [0])
    e.close()
    vl, edges, batches = _random_stream(31)
    eu = [a for a, _ in edges]
    ev = [b for _, b in edges]
    q = ([0, 1, 2, 0], [(0, 1), (1, 2), (2, 0), (2, 3)])
    e1, e2 = bd.Engine(vl, eu, ev), bd.Engine(vl, eu, ev)
    e1.add_query(*q)
    e2.add_query(*q)
    buf = bd.make_updates(batches[0])
    e2.submit_batch(buf)
    for bi, b in enumerate(batches):
        r1 = e1.match_batch(b)
        r2 = e2.wait()
        if bi + 1 < len(batches):
            e2.submit_batch(bd.make_updates(batches[bi + 1]))
        assert (r1.positive, r1.negative) == (r2.positive, r2.negative), bi
    for v in range(0, len(vl), 97):
        assert e1.neighbors(v) == e2.neighbors(v)
    e1.close()
    e2.close()


def test_multi_query_sums_and_independence():
    import paper_2401_17018_b200 as bd
    insts = gu.load("streams")[:6]
    for inst in insts:
        vl, eu, ev, el, ql, qe, batches = gu.instance_arrays(inst)
        e = bd.Engine(vl, eu, ev, el)
        e.add_query(ql, qe)
        e.add_query(ql, qe)  # same query twice: identical counts
        for b, exp in zip(batches, inst["expect"]):
            r = e.match_batch(b)
            assert r.positive == [exp["pos"]] * 2 and r.negative == [exp["neg"]] * 2


def test_rows_match_restatement():
    import paper_2401_17018_b200 as bd
    from oracle_py import Oracle
    for inst in gu.load("streams")[40:44]:
        vl, eu, ev, el, ql, qe, batches = gu.instance_arrays(inst)
        e = bd.Engine(vl, eu, ev, el)
        e.add_query(ql, qe)
        o = Oracle(vl, eu, ev, el)
        o.add_query(ql, qe)
        for b in batches:
            e.match_batch(b)
            o.apply_batch(b)
            rows = e.rows(0)
            assert all(int(rows[v]) == o.row(0, v) for v in range(len(vl)))
        # no replanning in either: the orders are the ones built at add_query
        assert [e.order(0, k) for k in range(len(qe))] == [o.order(0, k) for k in range(len(qe))]


@pytest.mark.parametrize("world", [2, 3])
def test_gpu_work_split_sums_to_reference(world):
    """Each engine counts only its share of the work units (multi-GPU split);
    run all shards on one GPU and sum."""
    import paper_2401_17018_b200 as bd
    insts = gu.load("streams")[-4:] + gu.load("skewed")
    for inst in insts:
        vl, eu, ev, el, ql, qe, batches = gu.instance_arrays(inst)
        engines = []
        for r in range(world):
            e = bd.Engine(vl, eu, ev, el, shard_rank=r, shard_world=world)
            e.add_query(ql, qe)
            engines.append(e)
        for b, exp in zip(batches, inst["expect"]):
            rs = [e.match_batch(b) for e in engines]
            assert sum(r.positive[0] for r in rs) == exp["pos"], inst["name"]
            assert sum(r.negative[0] for r in rs) == exp["neg"], inst["name"]


def _random_stream(seed, V=2500, E=20000, L=3, nb=12, bsz=300):
    import numpy as np
    rng = np.random.default_rng(seed)
    vl = rng.integers(0, L, V).astype(np.uint32)
    hubs = rng.integers(0, V, 20)
    pairs = set()
    while len(pairs) < E:
        a = int(hubs[rng.integers(0, 20)]) if rng.random() < 0.2 else int(rng.integers(0, V))
        b = int(rng.integers(0, V))
        if a != b:
            pairs.add((min(a, b), max(a, b)))
    present = set(pairs)
    edges = sorted(pairs)
    batches = []
    for _ in range(nb):
        batch, used = [], set()
        plist = sorted(present)
        while len(batch) < bsz:
            if rng.random() < 0.34:
                k = plist[int(rng.integers(0, len(plist)))]
                op = 1
            else:
                a, b = (int(x) for x in rng.integers(0, V, 2))
                k = (min(a, b), max(a, b))
                op = 0
                if a == b or k in present:
                    continue
            if k in used:
                continue
            used.add(k)
            batch.append((op, k[0], k[1]))
        for op, a, b in batch:
            (present.discard if op else present.add)((a, b))
        batches.append(batch)
    return vl, edges, batches


@pytest.mark.parametrize("opts", [{"zero_copy": True}, {"l2_hot_mb": 1}])
def test_storage_options_do_not_change_counts(opts):
    """Zero-copy adjacency pool (mapped pinned host memory) and K8 hot-list
    packing into an L2-persisting arena (every 8 batches, so batches 9-12 read
    packed lists) are storage/performance choices only: counts equal the
    CPU restatement (pinned to the reference) on every batch."""
    import sys
    import os
    import paper_2401_17018_b200 as bd
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
    from oracle_py import Oracle
    vl, edges, batches = _random_stream(11)
    eu = [a for a, _ in edges]
    ev = [b for _, b in edges]
    q = ([0, 1, 2, 0, 1], [(0, 1), (1, 2), (2, 0), (2, 3), (3, 4)])
    e = bd.Engine(vl, eu, ev, **opts)
    e.add_query(*q)
    o = Oracle(vl, eu, ev)
    o.add_query(*q)
    for bi, b in enumerate(batches):
        r = e.match_batch(b)
        exp = o.apply_batch(b)
        assert (r.positive[0], r.negative[0]) == (exp[0][0], exp[1][0]), (bi, opts)
    e.close()


def test_hub_bitmaps_do_not_change_counts(monkeypatch):
    """Membership bitmaps (normally for lists >= 1024) forced onto every
    vertex with >= 4 neighbours, so the golden suites run the bitmap
    membership tests and their maintenance by the merge."""
    monkeypatch.setenv("BDSM_BITMAP_MINDEG", "4")
    for suite in ("streams", "skewed", "matcher_random"):
        for inst in gu.load(suite):
            e, batches = _engine(inst)
            for bi, (b, exp) in enumerate(zip(batches, inst["expect"])):
                r = e.match_batch(b)
                assert (r.positive[0], r.negative[0]) == (exp["pos"], exp["neg"]), (suite, inst["name"], bi)
            e.close()


@pytest.mark.parametrize("self_scan", ["0", "1000000"])
def test_anchor_offset_scan_paths(monkeypatch, self_scan):
    """Anchor offsets come from a separate device scan (large batches) or from
    k_anchor_emit's own block scan (batches up to 16K updates); both paths,
    forced on every golden suite, give the reference's counts."""
    monkeypatch.setenv("BDSM_TUNE_SELFSCAN", self_scan)
    for suite in gu.SUITES:
        for inst in gu.load(suite):
            e, batches = _engine(inst)
            for bi, (b, exp) in enumerate(zip(batches, inst["expect"])):
                r = e.match_batch(b)
                assert (r.positive[0], r.negative[0]) == (exp["pos"], exp["neg"]), (suite, inst["name"], bi)
            e.close()


@pytest.mark.parametrize("small_group", ["1", "8", "16"])
@pytest.mark.parametrize("bitmap_mindeg", [None, "4"])
def test_thread_merge_matches_reference(monkeypatch, bitmap_mindeg, small_group):
    """Short lists (<= 256 entries) of large batches are merged one per lane
    group (k_merge_group, 8 or 16 lanes per list) or one per thread
    (k_merge_small); the threshold is lowered so every golden batch takes
    that path: counts equal the reference's, and on a mixed random stream
    every neighbour list equals the expected one after each batch.  With
    bitmaps forced onto small vertices the short-list path's bitmap
    maintenance is exercised too."""
    import os
    import sys
    import paper_2401_17018_b200 as bd
    monkeypatch.setenv("BDSM_TUNE_SMALLMIN", "1")
    monkeypatch.setenv("BDSM_TUNE_SMALL_GROUP", small_group)
    if bitmap_mindeg:
        monkeypatch.setenv("BDSM_BITMAP_MINDEG", bitmap_mindeg)
    for suite in gu.SUITES:
        for inst in gu.load(suite):
            e, batches = _engine(inst)
            for bi, (b, exp) in enumerate(zip(batches, inst["expect"])):
                r = e.match_batch(b)
                assert (r.positive[0], r.negative[0]) == (exp["pos"], exp["neg"]), (suite, inst["name"], bi)
            e.close()
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
    from oracle_py import Oracle
    vl, edges, batches = _random_stream(23)
    eu = [a for a, _ in edges]
    ev = [b for _, b in edges]
    q = ([0, 1, 2, 0], [(0, 1), (1, 2), (2, 0), (2, 3)])
    e = bd.Engine(vl, eu, ev)
    e.add_query(*q)
    o = Oracle(vl, eu, ev)
    o.add_query(*q)
    adj = {v: set() for v in range(len(vl))}
    for a, b in edges:
        adj[a].add(b)
        adj[b].add(a)
    for bi, b in enumerate(batches):
        r = e.match_batch(b)
        exp = o.apply_batch(b)
        assert (r.positive[0], r.negative[0]) == (exp[0][0], exp[1][0]), bi
        for op, x, y in b:
            (adj[x].discard if op else adj[x].add)(y)
            (adj[y].discard if op else adj[y].add)(x)
        for v in range(0, len(vl), 7):
            assert e.neighbors(v) == sorted(adj[v]), (bi, v)
    e.close()


def test_long_list_merge_matches_restatement():
    """Lists of >= 4096 entries are merged by a whole CTA (k_merge_big), in
    place (delete-only / insert-only) or relocated (mixed): a 5000-neighbour
    hub receiving inserts and deletes over several batches, checked against
    the CPU restatement batch by batch, plus its final neighbour list."""
    import os
    import sys
    import numpy as np
    import paper_2401_17018_b200 as bd
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
    from oracle_py import Oracle
    rng = np.random.default_rng(5)
    V, L = 7000, 3
    vl = rng.integers(0, L, V).astype(np.uint32)
    hub = 0
    pairs = {(0, v) for v in range(1, 5001)}
    while len(pairs) < 20000:
        a, b = (int(x) for x in rng.integers(1, V, 2))
        if a != b:
            pairs.add((min(a, b), max(a, b)))
    present = set(pairs)
    edges = sorted(pairs)
    q = ([0, 1, 2, 1], [(0, 1), (1, 2), (2, 0), (0, 3)])
    e = bd.Engine(vl, [a for a, _ in edges], [b for _, b in edges])
    e.add_query(*q)
    o = Oracle(vl, [a for a, _ in edges], [b for _, b in edges])
    o.add_query(*q)
    kinds = ["delete", "insert", "mixed", "mixed", "delete", "insert"]
    for bi, kind in enumerate(kinds):
        batch, used = [], set()
        hub_nb = sorted(b for a, b in present if a == hub)
        while len(batch) < 200:
            if kind == "delete" or (kind == "mixed" and len(batch) % 2):
                k = (hub, hub_nb[int(rng.integers(0, len(hub_nb)))])
                op = 1
            else:
                v = int(rng.integers(1, V))
                k = (hub, v)
                op = 0
                if k in present:
                    continue
            if k in used:
                continue
            used.add(k)
            batch.append((op, k[0], k[1]))
        for op, a, b in batch:
            (present.discard if op else present.add)((a, b))
        r = e.match_batch(batch)
        exp = o.apply_batch(batch)
        assert (r.positive[0], r.negative[0]) == (exp[0][0], exp[1][0]), (bi, kind)
    assert e.neighbors(hub) == sorted(b for a, b in present if a == hub)
    e.close()


@pytest.mark.parametrize("group_bits", [1, 3])
def test_group_bits_only_filter(group_bits):
    """--group-bits changes the NLF counter width (the candidate filter,
    src/encoding.cpp:17-24), never the counts (PipelineConfig::group_bits)."""
    import paper_2401_17018_b200 as bd
    for inst in gu.load("streams")[:20] + gu.load("fig1"):
        vl, eu, ev, el, ql, qe, batches = gu.instance_arrays(inst)
        e = bd.Engine(vl, eu, ev, el, group_bits=group_bits)
        e.add_query(ql, qe)
        for b, exp in zip(batches, inst["expect"]):
            r = e.match_batch(b)
            assert (r.positive[0], r.negative[0]) == (exp["pos"], exp["neg"]), (inst["name"], group_bits)
        e.close()


def test_deadline_marks_query_unsolved():
    """MatchOptions::deadline / --timeout (src/scheduler.cpp:101-110,
    src/bench.cpp:418-432): a query whose budget has run out is reported in
    stats.timed_out, its counts are dropped, and it is skipped afterwards;
    other queries are unaffected."""
    import time
    import paper_2401_17018_b200 as bd
    inst = gu.load("skewed")[0]
    vl, eu, ev, el, ql, qe, batches = gu.instance_arrays(inst)
    e = bd.Engine(vl, eu, ev, el)
    q0 = e.add_query(ql, qe)
    q1 = e.add_query(ql, qe)
    e.set_deadline(q0, 1e-9)
    time.sleep(0.01)
    r = e.match_batch(batches[0])
    assert r.stats["timed_out"] & (1 << q0)
    assert r.positive[q0] == 0 and r.negative[q0] == 0
    assert (r.positive[q1], r.negative[q1]) == (inst["expect"][0]["pos"], inst["expect"][0]["neg"])
    e.close()


@pytest.mark.parametrize("suite", gu.SUITES)
def test_exact_coalescing_equals_reference(suite):
    """Exact coalesced search: one anchored orientation per
    automorphism orbit of directed query edges, weighted by the orbit size;
    the counts must equal the reference's coalesce-off counts on every batch
    (the reference's own coalesced search misses matches, F1)."""
    for inst in gu.load(suite):
        e, batches = _engine(inst, coalesce=True)
        for bi, (b, exp) in enumerate(zip(batches, inst["expect"])):
            r = e.match_batch(b)
            assert (r.positive[0], r.negative[0]) == (exp["pos"], exp["neg"]), (inst["name"], bi)
        e.close()


def test_exact_coalescing_unlabelled_cliques_and_cycles():
    """Symmetric unlabelled queries (the C5 sweep shapes): coalesced == plain on
    a random mixed stream, with 20x / 10x fewer anchored searches."""
    import numpy as np
    import paper_2401_17018_b200 as bd
    rng = np.random.default_rng(11)
    V, E = 400, 6000
    pairs = set()
    while len(pairs) < E:
        a, b = (int(x) for x in rng.integers(0, V, 2))
        if a != b:
            pairs.add((min(a, b), max(a, b)))
    pairs = sorted(pairs)
    eu = np.array([p[0] for p in pairs], np.uint32)
    ev = np.array([p[1] for p in pairs], np.uint32)
    vl = np.zeros(V, np.uint32)
    queries = [[(i, j) for i in range(4) for j in range(i + 1, 4)],  # K4
               [(i, (i + 1) % 5) for i in range(5)],                 # C5
               [(0, 1), (1, 2), (2, 3), (3, 0), (0, 2)]]             # diamond
    plain = bd.Engine(vl, eu, ev)
    co = bd.Engine(vl, eu, ev, coalesce=True)
    o = Oracle(vl, eu, ev)
    for qe in queries:
        n = max(max(x) for x in qe) + 1
        plain.add_query([0] * n, qe)
        co.add_query([0] * n, qe)
        o.add_query([0] * n, qe)
    present = set(pairs)
    for _ in range(3):
        batch, used = [], set()
        while len(batch) < 60:
            if rng.random() < 0.4:
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
        rp, rc = plain.match_batch(batch), co.match_batch(batch)
        exp = o.apply_batch(batch)
        assert (rc.positive, rc.negative) == (rp.positive, rp.negative) == (exp[0], exp[1])
        assert rc.stats["tasks"] < rp.stats["tasks"]
        for op, a, b in batch:
            k = (min(a, b), max(a, b))
            (present.add if op == 0 else present.discard)(k)
    plain.close()
    co.close()

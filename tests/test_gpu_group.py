"""Multi-device engine group (bdsm_group_*, SURVEY.md §8(e) in one process):
every engine holds a replica and counts its share of the work units, and the
summed counts equal the reference's golden counts.  On the one-GPU box the
group's engines share device 0 (the split is exact whatever the devices)."""
import numpy as np
import pytest

import golden_util as gu

pytestmark = pytest.mark.gpu


def _group(inst, devices, **kw):
    import paper_2401_17018_b200 as bd
    vl, eu, ev, el, ql, qe, batches = gu.instance_arrays(inst)
    g = bd.EngineGroup(vl, eu, ev, el, devices=devices, **kw)
    g.add_query(ql, qe)
    return g, batches


@pytest.mark.parametrize("devices", [[0, 0], [0, 0, 0]])
@pytest.mark.parametrize("suite", ["skewed", "matcher_random", "edge_labeled", "streams"])
def test_group_counts_equal_reference(suite, devices):
    for inst in gu.load(suite):
        g, batches = _group(inst, devices)
        assert g.size == len(devices)
        for bi, (b, exp) in enumerate(zip(batches, inst["expect"])):
            r = g.match_batch(b)
            assert (r.positive[0], r.negative[0]) == (exp["pos"], exp["neg"]), (suite, inst["name"], bi)
        g.close()


def test_group_stream_and_replicas():
    import paper_2401_17018_b200 as bd
    for inst in gu.load("streams")[-6:]:
        g, batches = _group(inst, [0, 0, 0, 0])
        rs = g.match_stream(batches)
        assert [(r.positive[0], r.negative[0]) for r in rs] == [(x["pos"], x["neg"]) for x in inst["expect"]]
        # every replica holds the same graph after the stream
        vl, eu, ev, el, ql, qe, _ = gu.instance_arrays(inst)
        e = bd.Engine(vl, eu, ev, el)
        e.add_query(ql, qe)
        for b in batches:
            e.match_batch(b)
        for v in range(0, len(vl), max(1, len(vl) // 50)):
            want = e.neighbors(v)
            assert all(g.neighbors(v, r) == want for r in range(4)), (inst["name"], v)
        e.close()
        g.close()


def test_group_batch_error_all_or_nothing():
    import paper_2401_17018_b200 as bd
    fig = {i["name"]: i for i in gu.load("fig1")}
    g, _ = _group(fig["fig1_batch"], [0, 0])
    with pytest.raises(bd.BatchError) as ei:
        g.match_batch([(0, 0, 2), (1, 0, 1), (0, 0, 3), (0, 0, 99)])
    assert ei.value.failures == [(1, 3), (2, 2), (3, 1)]
    with pytest.raises(ValueError, match="self-loop update"):
        g.match_batch([(0, 0, 2), (0, 3, 3)])
    r = g.match_batch([(0, 0, 2), (0, 1, 4), (1, 4, 5)])  # nothing of the rejected batch was applied
    assert (r.positive, r.negative) == ([4], [0])
    g.close()


def test_group_matches_equal_single_engine():
    import paper_2401_17018_b200 as bd
    for inst in gu.load("matcher_random")[:20]:
        vl, eu, ev, el, ql, qe, batches = gu.instance_arrays(inst)
        e = bd.Engine(vl, eu, ev, el)
        e.add_query(ql, qe)
        e.collect_matches(1 << 16)
        g, _ = _group(inst, [0, 0, 0])
        g.collect_matches(1 << 16)
        for b in batches:
            e.match_batch(b)
            g.match_batch(b)
            for pos in (False, True):
                assert np.array_equal(g.matches(0, pos), e.matches(0, pos)), inst["name"]
        e.close()
        g.close()


def test_group_matches_cap():
    """More matches than the collect cap: the count is reported and the rows
    are refused (Engine.matches' contract), without fetching them."""
    import paper_2401_17018_b200 as bd
    fig = {i["name"]: i for i in gu.load("fig1")}
    g, _ = _group(fig["fig1_batch"], [0, 0])
    g.collect_matches(2)
    r = g.match_batch([(0, 0, 2), (0, 1, 4), (1, 4, 5)])
    assert r.positive == [4]
    with pytest.raises(bd.EngineError, match="4 matches"):
        g.matches(0, True)
    g.collect_matches(8)
    r = g.match_batch([(1, 0, 2)])  # deleting (0, 2) removes the matches through it
    assert len(g.matches(0, False)) == r.negative[0]
    g.close()


def test_engine_matches_cap():
    """Engine.matches refuses a truncated match set the same way."""
    import paper_2401_17018_b200 as bd
    fig = {i["name"]: i for i in gu.load("fig1")}
    vl, eu, ev, el, ql, qe, _ = gu.instance_arrays(fig["fig1_batch"])
    e = bd.Engine(vl, eu, ev, el)
    e.add_query(ql, qe)
    e.collect_matches(2)
    assert e.match_batch([(0, 0, 2), (0, 1, 4), (1, 4, 5)]).positive == [4]
    with pytest.raises(bd.EngineError, match="4 matches"):
        e.matches(0, True)
    e.close()

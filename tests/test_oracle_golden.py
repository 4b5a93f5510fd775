"""Pins the CPU restatement (oracle/) to the reference: on every golden
instance its counts equal the reference's match_batch (coalesce off) and the
brute-force oracle, and its dfs_visits / intersection_ops / tasks_run equal the
reference's MatchStats."""
import pytest

import golden_util as gu
from oracle_py import Oracle, OracleError


@pytest.mark.parametrize("suite", gu.SUITES)
def test_restatement_equals_reference(suite):
    for inst in gu.load(suite):
        vl, eu, ev, el, ql, qe, batches = gu.instance_arrays(inst)
        o = Oracle(vl, eu, ev, el)
        o.add_query(ql, qe)
        for b, exp in zip(batches, inst["expect"]):
            pos, neg, st = o.apply_batch(b)
            assert (pos[0], neg[0]) == (exp["pos"], exp["neg"]), inst["name"]
            if exp["brute_pos"] >= 0:
                assert (pos[0], neg[0]) == (exp["brute_pos"], exp["brute_neg"]), inst["name"]
            assert st[0] == exp["visits"], inst["name"]
            assert st[1] == exp["iops"], inst["name"]
            assert st[2] == exp["tasks"], inst["name"]


def test_threads_do_not_change_counts():
    inst = gu.load("skewed")[0]
    vl, eu, ev, el, ql, qe, batches = gu.instance_arrays(inst)
    o = Oracle(vl, eu, ev, el)
    o.add_query(ql, qe)
    pos, neg, st = o.apply_batch(batches[0], nthreads=4)
    assert pos == [400 * 120 + 3] and neg == [0]


def test_fig1_kats():
    fig = {i["name"]: i for i in gu.load("fig1")}
    vl, eu, ev, el, ql, qe, batches = gu.instance_arrays(fig["fig1_singletons"])
    o = Oracle(vl, eu, ev, el)
    o.add_query(ql, qe)
    got = [o.apply_batch(b)[:2] for b in batches]
    assert got == [([4], [0]), ([2], [0]), ([0], [2])]


def test_batch_errors_are_all_or_nothing():
    fig = {i["name"]: i for i in gu.load("fig1")}
    vl, eu, ev, el, ql, qe, _ = gu.instance_arrays(fig["fig1_batch"])
    o = Oracle(vl, eu, ev, el)
    o.add_query(ql, qe)
    with pytest.raises(OracleError) as ei:
        o.apply_batch([(0, 0, 2), (1, 0, 1), (0, 0, 3), (0, 0, 99)])
    assert ei.value.status == 1
    assert ei.value.failures == [(1, 3), (2, 2), (3, 1)]
    # nothing applied: the real batch still gives the documented +4/-0
    assert o.apply_batch([(0, 0, 2), (0, 1, 4), (1, 4, 5)])[:2] == ([4], [0])
    with pytest.raises(OracleError) as ei:
        o.apply_batch([(0, 3, 3)])
    assert ei.value.status == 2
    with pytest.raises(OracleError) as ei:
        o.apply_batch([(0, 1, 7), (1, 7, 1)])
    assert ei.value.status == 2

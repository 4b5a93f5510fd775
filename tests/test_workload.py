"""The synthetic workload generators (bench infrastructure): deterministic,
shape properties of SURVEY.md §8(d), every batch valid against the evolving
graph (the restatement applies them without BatchError), and the binary
workload file round-trips through the C++ reader used by the CPU baselines."""
import json
import os
import subprocess

import numpy as np

import workload as W

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ops(b):
    return [(int(x["op"]), int(x["u"]), int(x["v"])) for x in b]


def test_c2_shape_and_validity():
    from oracle_py import Oracle
    wl = W.build("C2", 3, scale_down=100, device="cpu", batch=1500)
    m = wl.meta
    assert m["E"] == 690_000 and m["V"] == 48_000 and m["isolated"] == 0
    assert m["d_max"] <= 1.5 * 200  # expected-degree cap dmax/scale_down; realised degrees fluctuate
    keys = np.minimum(wl.src, wl.dst).astype(np.uint64) << 32 | np.maximum(wl.src, wl.dst)
    assert len(np.unique(keys)) == len(keys) and np.all(wl.src != wl.dst)
    assert len(wl.qlabels) == 6 and len(wl.qedges) >= 6 and 2 * len(wl.qedges) / 6 < 3  # sparse, with a cycle
    o = Oracle(wl.labels, wl.src, wl.dst)
    o.add_query(wl.qlabels, wl.qedges)
    emitted = 0
    for b in wl.batches:
        ops = b["op"]
        assert np.array_equal(ops, ((np.arange(len(b)) + emitted) % 3 == 2).astype(np.uint32))
        emitted += len(b)
        pk = np.minimum(b["u"], b["v"]).astype(np.uint64) << 32 | np.maximum(b["u"], b["v"])
        assert len(np.unique(pk)) == len(pk)
        o.apply_batch(_ops(b), match=False)  # raises on any invalid update


def test_rmat_c1_shape():
    wl = W.build("C1", 1, device="cpu")
    assert wl.V == 65536 and len(wl.src) == 1_000_000
    assert 8000 < wl.meta["d_max"] < 13000  # ~10.3K at s16
    assert 0.2 < wl.meta["isolated"] / wl.V < 0.35  # ~27 % isolated
    assert np.all(wl.batches[0]["op"] == 0) and len(wl.batches[0]) == 1000


def test_deterministic():
    a = W.build("C2", 2, scale_down=200, device="cpu", batch=500)
    b = W.build("C2", 2, scale_down=200, device="cpu", batch=500)
    assert np.array_equal(a.src, b.src) and np.array_equal(a.labels, b.labels)
    assert a.qedges == b.qedges and all(np.array_equal(x, y) for x, y in zip(a.batches, b.batches))


def test_workload_file_round_trip(tmp_path):
    from oracle_py import Oracle, build
    build()
    wl = W.build("C2", 2, scale_down=200, device="cpu", batch=600)
    path = str(tmp_path / "w.bin")
    W.write_file(wl, path)
    out = subprocess.run([os.path.join(REPO, "oracle", "oracle_bench"), path, "--threads", "2"],
                         capture_output=True, text=True, check=True).stdout
    lines = [json.loads(l) for l in out.splitlines() if l.startswith("{")]
    per = [l for l in lines if "batch" in l]
    o = Oracle(wl.labels, wl.src, wl.dst)
    o.add_query(wl.qlabels, wl.qedges)
    for b, l in zip(wl.batches, per):
        pos, neg, _ = o.apply_batch(_ops(b), nthreads=2)
        assert (l["positive"], l["negative"]) == (pos[0], neg[0])

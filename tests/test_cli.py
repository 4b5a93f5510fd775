"""`bdsm run` CLI drop-in (reference tools/bdsm.cpp:26-156) against fixtures
produced by the reference's own `bdsm run` path (tests/golden/make_cli_golden.py,
oracle/ref_cli.cpp: run_pipeline with coalesce off).

CPU: the seeded generators (`bdsm generate`) reproduce the reference's
generate_queries / generate_stream byte for byte; flag errors.
GPU: `bdsm run` writes the reference's deltas.csv, summary line and
--dump-matches files, and the report CSV headers of emit_report
(src/bench.cpp:566-591).
"""
import json
import os
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(REPO, "paper_2401_17018_b200", "bdsm")
GOLD = os.path.join(REPO, "tests", "golden", "cli")
CASES = sorted(d for d in os.listdir(GOLD) if os.path.exists(os.path.join(GOLD, d, "case.json")))
GEN_CASES = [c for c in CASES if c.startswith("gen_")]


def case(name):
    with open(os.path.join(GOLD, name, "case.json")) as f:
        return json.load(f)


def cli_args(name, meta, out):
    d = os.path.join(GOLD, name)
    graph = os.path.join(d, "g.txt")
    q, s = meta["qspec"], meta["sspec"]
    args = []
    if q.startswith("q:"):
        args += ["--query", os.path.join(GOLD, q[2:])]
        graph = os.path.join(GOLD, os.path.dirname(q[2:]), "g.txt")
    else:
        args += ["--gen-queries", q[2:]]
    sv = s[2:]
    if "," in sv:
        args += ["--gen-stream", sv]
    else:
        args += ["--stream", os.path.join(GOLD, sv)]
    return ["--graph", graph] + args + ["--seed", str(meta["seed"]), "--out", out]


def read(p):
    with open(p) as f:
        return f.read()


def test_cli_built():
    assert os.access(CLI, os.X_OK), "build the CLI: bash paper_2401_17018_b200/build.sh"


@pytest.mark.parametrize("name", GEN_CASES)
def test_generators_match_reference(name, tmp_path):
    meta = case(name)
    out = str(tmp_path / "gen")
    r = subprocess.run([CLI, "generate"] + cli_args(name, meta, out), capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    ref = os.path.join(GOLD, name, "ref")
    files = sorted(f for f in os.listdir(ref) if f.startswith("query_") or f == "stream.txt")
    assert files and sorted(f for f in os.listdir(out)) == files
    for f in files:
        assert read(os.path.join(out, f)) == read(os.path.join(ref, f)), f


def test_cli_errors(tmp_path):
    r = subprocess.run([CLI], capture_output=True, text=True)
    assert r.returncode != 0
    r = subprocess.run([CLI, "run", "--graph", "x", "--bogus", "1"], capture_output=True, text=True)
    assert r.returncode != 0 and "--bogus" in r.stderr
    g = os.path.join(GOLD, "fig1", "g.txt")
    r = subprocess.run([CLI, "run", "--graph", g, "--query", g, "--stream", g, "--stealing", "sometimes"],
                       capture_output=True, text=True)
    assert r.returncode == 1 and r.stderr.startswith("error: unknown stealing mode"), r.stderr
    r = subprocess.run([CLI, "generate", "--graph", str(tmp_path / "missing.txt")], capture_output=True, text=True)
    assert r.returncode == 1 and "error: cannot open" in r.stderr
    bad = tmp_path / "bad.txt"
    bad.write_text("v 0 1\nx 1 2\n")
    r = subprocess.run([CLI, "generate", "--graph", str(bad)], capture_output=True, text=True)
    assert r.returncode == 1 and "unknown record 'x' at line 2" in r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_cli_run_matches_reference(name, tmp_path):
    meta = case(name)
    out = str(tmp_path / "out")
    dump = ["--dump-matches"] if meta.get("dump_matches") else []
    r = subprocess.run([CLI, "run"] + cli_args(name, meta, out) + dump, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip() == meta["summary"].replace("OUT/", out + "/")
    ref = os.path.join(GOLD, name, "ref")
    assert read(os.path.join(out, "deltas.csv")) == read(os.path.join(ref, "deltas.csv"))
    # --dump-matches: the materialised match sets, file for file (src/bench.cpp:484-491)
    dumps = sorted(f for f in os.listdir(ref) if f.startswith("matches_batch"))
    assert bool(dumps) == bool(dump)
    for f in dumps:
        assert read(os.path.join(out, f)) == read(os.path.join(ref, f)), f
    assert read(os.path.join(out, "latency.csv")).startswith("query_id,category,size,seconds,solved\n")
    assert read(os.path.join(out, "stages.csv")).startswith("batch,preprocess_s,match_s,ratio\n")
    assert read(os.path.join(out, "utilization.csv")).startswith("worker,busy_seconds,total_seconds,fraction\n")


@pytest.mark.gpu
def test_cli_batch_error(tmp_path):
    g = os.path.join(GOLD, "fig1", "g.txt")
    q = os.path.join(GOLD, "fig1", "q.txt")
    s = tmp_path / "s.txt"
    s.write_text("+ 0 3\n")  # (0,3) exists: BatchError, CLI prints error and exits 1
    r = subprocess.run([CLI, "run", "--graph", g, "--query", q, "--stream", str(s), "--out", str(tmp_path / "o")],
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 1 and r.stderr.startswith("error: batch rejected: 1 invalid update(s)"), r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["gen_sparse_mixed", "gen_sparse50_mixed", "gen_dense_delete", "fig1_s3"])
def test_cli_exact_coalescing_matches_reference(name, tmp_path):
    """`--coalesce on` runs the exact coalesced search: the reference's
    coalesce-off deltas (the reference's own coalesced search misses matches)."""
    meta = case(name)
    out = str(tmp_path / "out")
    r = subprocess.run([CLI, "run"] + cli_args(name, meta, out) + ["--coalesce", "on"], capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip() == meta["summary"].replace("OUT/", out + "/")
    assert read(os.path.join(out, "deltas.csv")) == read(os.path.join(GOLD, name, "ref", "deltas.csv"))


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_cli_multi_device_group_matches_reference(name, tmp_path):
    """`--devices 0,0,0`: a multi-device group (replicas, work units split over
    three engines sharing the one GPU) writes the reference's deltas and match
    dumps."""
    meta = case(name)
    out = str(tmp_path / "out")
    dump = ["--dump-matches"] if meta.get("dump_matches") else []
    r = subprocess.run([CLI, "run"] + cli_args(name, meta, out) + dump + ["--devices", "0,0,0"], capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip() == meta["summary"].replace("OUT/", out + "/")
    ref = os.path.join(GOLD, name, "ref")
    assert read(os.path.join(out, "deltas.csv")) == read(os.path.join(ref, "deltas.csv"))
    for f in sorted(f for f in os.listdir(ref) if f.startswith("matches_batch")):
        assert read(os.path.join(out, f)) == read(os.path.join(ref, f)), f

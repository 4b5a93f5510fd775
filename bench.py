#!/usr/bin/env python
"""Benchmark of the per-batch hot path (match_batch) — prints ONE JSON line.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

A step is one batch of the configured stream applied to the evolving graph:
validate -> negative phase on G -> merge + refresh -> positive phase on G'
-> counts.  Default workload: BASELINE.json configs[1]
(C2, LiveJournal-shaped, 6-vertex query, 10K mixed updates per batch).

  value   updates/s with the batch already resident in HBM (device-input
          C ABI entry point), device time from CUDA events on the engine's
          stream, max over ranks; L2 flushed between steps (outside timing).
  e2e     same metric through the host-buffer C ABI call (H2D of the batch
          and D2H of the counts inside the timed region), on a second engine
          replaying the same stream; its counts must equal the first's.
  roofline  dominant kernel's algorithmic bytes / its
          CUDA-event time vs MEASURED_PEAKS.json hbm_gbs.
  cpu_baseline  the UNMODIFIED reference (oracle/_ref/ref_bench) on a bounded
          prefix sample of the same stream, all host threads (rank 0, N=1).

--impl reference times the reference's own CPU path (oracle/_ref/ref_bench,
else the oracle port) on the same workload and prints the same line shape.
Multi-GPU (torchrun): graph replicated per rank, each batch's work units
split by the cost-balanced rule, counts summed with an NCCL all-reduce.
"""
from __future__ import annotations

import argparse
import json
import os
import shutil
import statistics
import subprocess
import sys
import tempfile
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workload as W  # noqa: E402

METRIC = "ms per update batch & updates/s (incremental matches), LJ-shape 6-vertex query"


def log(*a):
    print("[bench]", *a, file=sys.stderr, flush=True)


def peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.idx = device_index
        self.proc = None
        self.out = None

    def __enter__(self):
        if shutil.which("nvidia-smi"):
            self.out = tempfile.NamedTemporaryFile("w+", delete=False, suffix=".csv")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=self.out, stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.2)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.out:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        with open(self.out.name) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.out.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def run_reference_binary(path: str, prefix: int, batches: int, time_cap: float, timeout: float):
    """Runs oracle/_ref/ref_bench (else oracle/oracle_bench) on a workload file."""
    ref = os.path.join(REPO, "oracle", "_ref", "ref_bench")
    kind = "reference"
    if not os.path.exists(ref):
        subprocess.run(["make", "-s", "-C", os.path.join(REPO, "oracle")], check=False)
        ref = os.path.join(REPO, "oracle", "oracle_bench")
        kind = "port"
    cores = os.cpu_count() or 1
    flag = "--workers" if kind == "reference" else "--threads"
    cmd = [ref, path, flag, str(cores), "--prefix", str(prefix), "--batches", str(batches),
           "--time-cap", str(time_cap)]
    log("cpu baseline:", " ".join(cmd))
    t0 = time.time()
    try:
        out = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout)
        lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    except subprocess.TimeoutExpired as e:
        lines = [json.loads(l) for l in (e.stdout or b"").decode().splitlines() if l.startswith("{")]
        return {"kind": kind, "cores": cores, "error": f"timeout after {timeout:.0f}s", "batches": lines[:-1]}
    wall = time.time() - t0
    summ = [l for l in lines if l.get("summary")]
    per = [l for l in lines if "batch" in l]
    if not summ:
        return {"kind": kind, "cores": cores, "error": (out.stderr or out.stdout)[-300:], "batches": per}
    return {"kind": kind, "cores": cores, "summary": summ[0], "batches": per, "wall_s": wall}


def run_restatement_full(path: str, batches: int, timeout: float):
    """Full-batch parity checker: the CPU restatement (oracle/oracle_bench,
    pinned to the reference on tests/golden/ by counts and MatchStats) over the
    first `batches` complete batches of a workload file, all host threads."""
    exe = os.path.join(REPO, "oracle", "oracle_bench")
    if not os.path.exists(exe):
        subprocess.run(["make", "-s", "-C", os.path.join(REPO, "oracle")], check=False)
    cores = os.cpu_count() or 1
    cmd = [exe, path, "--threads", str(cores), "--batches", str(batches)]
    log("full-batch parity:", " ".join(cmd))
    t0 = time.time()
    try:
        out = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout)
        text = out.stdout
    except subprocess.TimeoutExpired as e:
        text = e.stdout.decode() if isinstance(e.stdout, bytes) else (e.stdout or "")
    lines = [json.loads(l) for l in text.splitlines() if l.startswith("{")]
    per = [l for l in lines if "batch" in l]
    summ = [l for l in lines if l.get("summary")]
    return {"batches": per, "summary": summ[0] if summ else None, "cores": cores, "wall_s": time.time() - t0}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def so_sha():
    """Build identity of the engine: a hash of its sources and build script
    (nvcc's fatbinaries embed temporary names, so the .so bytes differ between
    two builds of the same sources)."""
    import glob
    import hashlib
    h = hashlib.sha256()
    pkg = os.path.join(REPO, "paper_2401_17018_b200")
    files = sorted(glob.glob(os.path.join(pkg, "csrc", "*"))) + [os.path.join(pkg, "build.sh"),
                                                                   os.path.join(REPO, "include", "bdsm_gpu.h")]
    for f in files:
        h.update(os.path.basename(f).encode())
        with open(f, "rb") as fh:
            h.update(fh.read())
    return "src-" + h.hexdigest()[:16]


def physical_roofline(config, mk, mg, bker, bphase_ref, bupd, peak, peak_kind, step_ms, batch):
    """Roofline of the dominant kernel (k_wbm) from PHYSICAL bytes: the DRAM
    traffic per step of its launches in the committed ncu metrics capture of
    this build (profiles/traffic_<config>.json, tools/ncu_traffic.py) over its
    live CUDA-event time per step.  SURVEY.md §8(d)'s algorithmic figures (4 B
    per element of every backward list of a GenCandidates call) are reported
    beside it as equivalents: the kernel reads label sub-ranges, bitmap words
    and memoised weights, not whole lists, so those exceed any physical roof."""
    prof = os.path.join("profiles", f"traffic_{config.lower()}.json")
    tr, sha = None, so_sha()
    try:
        with open(os.path.join(REPO, prof)) as f:
            tr = json.load(f)
    except (OSError, ValueError):
        pass
    roof = {"bound": "hbm", "kernel": "k_wbm (K6 matching, negative + positive launch per step)", "peak": peak,
            "unit": "GB/s", "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)",
            "ms_per_step_live": mk, "share_of_step": mk / step_ms if step_ms else None,
            "algorithmic_equivalent": {
                "bytes_kernel_per_step": bker,
                "bytes_kernel_equivalent_GBps": bker / (mk / 1e3) / 1e9 if mk > 0 else 0.0,
                "reference_tree_bytes_per_step": bphase_ref,
                "reference_tree_equivalent_GBps": bphase_ref / (mk / 1e3) / 1e9 if mk > 0 else 0.0,
                "note": "SURVEY.md §8(d): 4 B x backward-list degrees per GenCandidates call, on the calls the "
                        "kernel makes (bytes_kernel) and on the reference DFS tree (B_phase); not physical"}}
    w = tr["kernels"].get("k_wbm") if tr else None
    if w:
        dram = w["dram_bytes_per_step"]
        achieved = dram / (mk / 1e3) / 1e9 if mk > 0 else 0.0
        roof.update({
            "achieved": achieved, "frac": achieved / peak,
            "traffic": dram / max(w["launches_per_step"], 1), "traffic_per_step": dram,
            "traffic_source": f"{prof}: dram__bytes_read.sum + dram__bytes_write.sum of the step's k_wbm launches "
                              f"(ncu metrics pass, build {tr.get('build')}, this build {sha}, "
                              f"{'same' if tr.get('build') == sha else 'DIFFERENT'} build)",
            "ncu_ms_per_step": w["ms_per_step"], "frac_at_ncu_time": w["dram_GBps"] / peak,
            "l2": {"bytes_per_step": w["l2_bytes_per_step"],
                   "achieved_GBps": w["l2_bytes_per_step"] / (mk / 1e3) / 1e9 if mk > 0 else 0.0,
                   "note": "lts__t_bytes.sum (all L2 traffic) of the same launches over the live time: the "
                           "re-read working set is L2-resident, the kernel is bound by dependent L2 round trips"},
        })
        m = tr["kernels"]
        merge = {k: m[k] for k in ("k_alloc", "k_merge_refresh", "k_merge_small", "k_merge_group", "k_merge_big",
                                   "k_finish_big")
                 if k in m}
        if merge:
            md = sum(v["dram_bytes_per_step"] for v in merge.values())
            roof["merge"] = {"kernels": sorted(merge), "dram_bytes_per_step": md, "b_upd_per_step": bupd,
                             "dram_over_b_upd": md / bupd if bupd else None, "ms_per_step_live": mg,
                             "dram_GBps_live": md / (mg / 1e3) / 1e9 if mg > 0 else 0.0}
    else:
        achieved = bker / (mk / 1e3) / 1e9 if mk > 0 else 0.0
        roof.update({"achieved": achieved, "frac": achieved / peak, "traffic": None,
                     "traffic_source": f"no ncu capture at {prof}: achieved is the algorithmic bytes_kernel "
                                       "figure, not physical"})
    return roof


def spawn_ranks(n: int) -> int:
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    log("spawning", n, "ranks:", " ".join(cmd))
    return subprocess.run(cmd).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--batch", type=int, default=None, help="override updates per batch")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-prefix", type=int, default=100, help="updates per CPU-baseline sub-batch")
    ap.add_argument("--cpu-batches", type=int, default=3)
    ap.add_argument("--cpu-time-cap", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--parity-full", type=int, default=-1,
                    help="batches checked against the CPU restatement at full size (-1: all; 0: off)")
    ap.add_argument("--parity-timeout", type=float, default=600.0)
    ap.add_argument("--chunk", type=int, default=32)
    ap.add_argument("--no-stream", action="store_true",
                    help="time one apply per batch instead of the pipelined stream")
    ap.add_argument("--coalesce", action="store_true", help="exact coalesced search (counts unchanged)")
    ap.add_argument("--l2-hot-mb", type=int, default=0, help="K8 hot-list L2 persistence budget (0: off)")
    args = ap.parse_args()

    world, rank, local = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # plain `python bench.py --gpus N`: start the N ranks here (one process
        # per GPU, torch.distributed.run on 127.0.0.1) and relay rank 0's line
        return spawn_ranks(args.gpus)
    if args.steps < 1 or args.warmup < 3:
        log("warmup must be >= 3 and steps >= 1")
    ndev = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if ndev:
        # more ranks than GPUs (functional test of the split on a 1-GPU box):
        # ranks share devices and the counts go through gloo
        local = local % ndev
    if world > 1:
        import torch.distributed as dist
        backend = "nccl" if ndev >= world else "gloo"
        if ndev:
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
    if args.impl == "reference":
        return reference_arm(args, world, rank)
    return ours(args, world, rank, local)


def gen_workload(args, nbatches, device):
    t0 = time.time()
    wl = W.build(args.config, nbatches, device=device, batch=args.batch)
    log(f"workload {args.config}: {wl.meta} query labels={wl.qlabels} edges={wl.qedges} "
        f"gen {time.time() - t0:.1f}s")
    return wl


def config_dict(args, wl, world):
    m = wl.meta
    return {"workload": f"{args.config}: {m['desc']}", "config_id": args.config, "V": m["V"], "E": m["E"],
            "labels": m["L"], "generator": m["generator"], "d_max": m["d_max"], "batch_updates": m["batch"],
            "batch_mode": m["mode"], "query_vertices": len(wl.qlabels), "query_edges": len(wl.qedges),
            "query_labels": wl.qlabels, "query": wl.qedges, "seeds": m["seeds"],
            "l2": ("pipelined stream: no flush between its batches, the graph (adjacency pool > 1 GB) exceeds the "
                   "126 MB L2; per-batch latency runs flush L2 (256 MiB write) before every batch"
                   if not getattr(args, "no_stream", False) else
                   "flushed (256 MiB write) before every timed step"),
            "parallelism": f"replicated graph, work units split over {world} GPU(s)" if world > 1 else "1 GPU",
            "coalesce": "exact (one search per automorphism orbit of directed query edges)" if args.coalesce
                        else "off"}


def reference_arm(args, world, rank):
    if rank != 0:
        return 0
    nb = max(args.steps + args.warmup, 1)
    device = "cuda" if torch.cuda.is_available() else "cpu"
    wl = gen_workload(args, nb, device)
    tmp = tempfile.mkdtemp(prefix="bdsm_ref_")
    path = os.path.join(tmp, "workload.bin")
    W.write_file(wl, path)
    steps = args.steps
    res = run_reference_binary(path, args.cpu_prefix, steps, time_cap=max(args.cpu_time_cap, 1.0) * 3,
                               timeout=900)
    shutil.rmtree(tmp, ignore_errors=True)
    line = {"impl": "reference", "metric": METRIC, "unit": "updates/s", "higher_is_better": True,
            "n_gpus": world, "steps": steps, "warmup": 0, "dtype": "u32", "data": "synthetic",
            "config": config_dict(args, wl, 1), "vs_baseline": None}
    if "summary" not in res:
        line.update({"value": None, "unavailable": res.get("error", "reference failed")})
    else:
        s = res["summary"]
        line.update({"value": s["updates_per_s"], "ms_per_step": s["median_ms"], "steps": s["batches"],
                     "cpu_baseline": {"value": s["updates_per_s"], "unit": "updates/s", "cores": res["cores"],
                                      "kind": res["kind"],
                                      "sample": f"first {args.cpu_prefix} updates of each of {s['batches']} "
                                                f"consecutive {wl.meta['batch']}-update batches (rest applied "
                                                f"untimed); graph build {s.get('build_s', 0):.1f}s excluded"},
                     "e2e": {"value": s["updates_per_s"], "unit": "updates/s", "h2d_bytes_per_step": 0,
                             "d2h_bytes_per_step": 0},
                     "per_batch": [{k: b[k] for k in ("positive", "negative", "ms", "dfs_visits")}
                                   for b in res["batches"]]})
    print(json.dumps(line), flush=True)
    return 0


def ours(args, world, rank, local):
    import paper_2401_17018_b200 as bd
    if not torch.cuda.is_available():
        print(json.dumps({"metric": METRIC, "error": "no CUDA device"}), flush=True)
        return 1
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    nb = args.warmup + args.steps
    wl = gen_workload(args, nb, dev)
    torch.cuda.synchronize()

    t0 = time.time()
    engA = bd.Engine(wl.labels, wl.src, wl.dst, device=local, shard_rank=rank, shard_world=world,
                     chunk=args.chunk, l2_hot_mb=args.l2_hot_mb, coalesce=args.coalesce)
    engA.add_query(wl.qlabels, wl.qedges)
    engB = bd.Engine(wl.labels, wl.src, wl.dst, device=local, shard_rank=rank, shard_world=world,
                     chunk=args.chunk, l2_hot_mb=args.l2_hot_mb, coalesce=args.coalesce)
    engB.add_query(wl.qlabels, wl.qedges)
    # pipelined stream: A and B run the timed batches as one stream, L (one
    # GPU) replays them one batch at a time for the per-batch latency (graphs
    # whose adjacency fits L2 are timed one flushed batch at a time)
    pipelined = not args.no_stream and 8 * wl.meta["E"] >= (256 << 20)
    args.no_stream = not pipelined
    engL = None
    if pipelined and world == 1:
        engL = bd.Engine(wl.labels, wl.src, wl.dst, device=local, chunk=args.chunk, l2_hot_mb=args.l2_hot_mb,
                         coalesce=args.coalesce)
        engL.add_query(wl.qlabels, wl.qedges)
    log(f"engines built in {time.time() - t0:.1f}s")

    # batches resident in HBM for `value`; pinned host copies for `e2e` (the
    # contract's host inputs are page-locked: the engine DMAs them directly)
    dev_batches = [torch.from_numpy(b.view(np.uint32).reshape(-1, 4).copy()).to(dev) for b in wl.batches]
    pinned_batches, pinned_keep = [], []
    for b in wl.batches:
        t = torch.empty(b.nbytes, dtype=torch.uint8, pin_memory=True)
        t.numpy()[:] = b.view(np.uint8)
        pinned_keep.append(t)
        pinned_batches.append(t.numpy().view(b.dtype))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    torch.cuda.synchronize()

    def allreduce(vals, op="sum"):
        if world == 1:
            return vals
        import torch.distributed as dist
        on = dev if dist.get_backend() == "nccl" else "cpu"
        t = torch.tensor(vals, dtype=torch.float64 if op == "max" else torch.int64, device=on)
        dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
        return t.tolist()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    # warm-up (every engine walks the same stream; the stream engines through
    # the stream call itself, so its buffers and kernels are in place)
    countsA, countsB, countsC = [], [], []
    if pipelined:
        for r in engA.match_stream_device([dev_batches[i].data_ptr() for i in range(args.warmup)],
                                          [len(wl.batches[i]) for i in range(args.warmup)]):
            countsA.append((r.positive[0], r.negative[0]))
        for r in engB.match_stream([pinned_batches[i] for i in range(args.warmup)]):
            countsB.append((r.positive[0], r.negative[0]))
    for i in range(args.warmup):
        if not pipelined:
            rA = engA.match_batch_device(dev_batches[i].data_ptr(), len(wl.batches[i]))
            rB = engB.match_batch(wl.batches[i])
            countsA.append((rA.positive[0], rA.negative[0]))
            countsB.append((rB.positive[0], rB.negative[0]))
        if engL:
            rC = engL.match_batch_device(dev_batches[i].data_ptr(), len(wl.batches[i]))
            countsC.append((rC.positive[0], rC.negative[0]))

    statsA = []
    dev_ms = []
    nccl_totals = []
    use_nccl = world > 1 and __import__("torch.distributed").distributed.get_backend() == "nccl"
    statsC, e2e_ms = [], []
    with ClockSampler(local if not os.environ.get("CUDA_VISIBLE_DEVICES") else 0) as clk:
        if pipelined:
            # per-batch latency: one apply per batch, L2 flushed before each
            for i in range(args.warmup, nb) if engL else []:
                flush.zero_()
                torch.cuda.synchronize()
                r = engL.match_batch_device(dev_batches[i].data_ptr(), len(wl.batches[i]))
                statsC.append(r.stats)
                countsC.append((r.positive[0], r.negative[0]))
            # value: the timed batches as one pipelined stream from HBM
            # (bdsm_engine_apply_stream); the graph (> 1 GB) exceeds L2
            flush.zero_()
            barrier()
            if use_nccl:
                # multi-GPU stream: NCCL broadcast of the
                # timed batches from rank 0, every rank streams them through its
                # replica counting its share of the work units, NCCL all-reduce
                # of the counts; CUDA events around all of it, max over ranks
                import torch.distributed as dist
                ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                ev0.record()
                for i in range(args.warmup, nb):
                    dist.broadcast(dev_batches[i].view(torch.int32), src=0)
                torch.cuda.current_stream().synchronize()
            rs = engA.match_stream_device([dev_batches[i].data_ptr() for i in range(args.warmup, nb)],
                                          [len(wl.batches[i]) for i in range(args.warmup, nb)])
            for r in rs:
                dev_ms.append(r.stats["ms_device"])
                statsA.append(r.stats)
                countsA.append((r.positive[0], r.negative[0]))
            if use_nccl:
                cnt = torch.tensor([c for r in rs for c in (r.positive[0], r.negative[0])], dtype=torch.int64,
                                   device=dev)
                dist.all_reduce(cnt)
                ev1.record()
                ev1.synchronize()
                total = ev0.elapsed_time(ev1)
                dev_ms = [total / args.steps] * args.steps
                nccl_totals.extend(tuple(x) for x in cnt.view(-1, 2).tolist())
            # e2e: the same stream through the C ABI with page-locked host
            # batches: every batch's H2D and its counts' D2H in the timed region
            flush.zero_()
            barrier()
            t1 = time.perf_counter()
            rs = engB.match_stream([pinned_batches[i] for i in range(args.warmup, nb)])
            e2e_total = (time.perf_counter() - t1) * 1e3
            e2e_ms = [e2e_total / args.steps] * args.steps
            for r in rs:
                countsB.append((r.positive[0], r.negative[0]))
        for i in range(args.warmup, nb) if not pipelined else []:
            flush.zero_()
            barrier()
            if use_nccl:
                # multi-GPU step: NCCL broadcast of the batch
                # from rank 0, each rank applies it to its replica and counts its
                # share of the work units, NCCL all-reduce of the counts; device
                # time from CUDA events around the whole step
                import torch.distributed as dist
                ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                ev0.record()
                dist.broadcast(dev_batches[i].view(torch.int32), src=0)
                torch.cuda.current_stream().synchronize()
                r = engA.match_batch_device(dev_batches[i].data_ptr(), len(wl.batches[i]))
                cnt = torch.tensor([r.positive[0], r.negative[0]], dtype=torch.int64, device=dev)
                dist.all_reduce(cnt)
                ev1.record()
                ev1.synchronize()
                dev_ms.append(ev0.elapsed_time(ev1))
                statsA.append(r.stats)
                countsA.append((r.positive[0], r.negative[0]))  # this rank's share
                nccl_totals.append(tuple(cnt.tolist()))
                continue
            r = engA.match_batch_device(dev_batches[i].data_ptr(), len(wl.batches[i]))
            dev_ms.append(r.stats["ms_device"])
            statsA.append(r.stats)
            countsA.append((r.positive[0], r.negative[0]))
        for i in range(args.warmup, nb) if not pipelined else []:
            flush.zero_()
            barrier()
            t1 = time.perf_counter()
            r = engB.match_batch(pinned_batches[i])
            e2e_ms.append((time.perf_counter() - t1) * 1e3)
            countsB.append((r.positive[0], r.negative[0]))
    barrier()
    clocks = clk.summary()

    tot_dev = allreduce([sum(dev_ms)], "max")[0]
    tot_e2e = allreduce([sum(e2e_ms)], "max")[0]
    flatA = allreduce([c for pn in countsA for c in pn])
    flatB = allreduce([c for pn in countsB for c in pn])
    if rank != 0:
        return 0
    updates = sum(len(b) for b in wl.batches[args.warmup:])
    value = updates / (tot_dev / 1e3)
    e2e_value = updates / (tot_e2e / 1e3)
    parity_ok = flatA == flatB and (not countsC or [c for pn in countsC for c in pn] == flatA)
    if nccl_totals:  # the in-step NCCL all-reduce agrees with the end-of-run sum
        parity_ok = parity_ok and [c for pn in nccl_totals for c in pn] == flatA[2 * args.warmup:]

    # roofline of the dominant kernel (mean over the timed steps)
    peak, peak_kind = peaks()
    mk = statistics.mean(s["ms_match_kernel"] for s in statsA)
    mg = statistics.mean(s["ms_merge_kernel"] for s in statsA)
    bker = statistics.mean(s["bytes_kernel"] for s in statsA)
    bphase_ref = statistics.mean(s["bytes_phase"] for s in statsA)
    bupd = statistics.mean(s["bytes_update"] for s in statsA)
    roof = physical_roofline(args.config, mk, mg, bker, bphase_ref, bupd, peak, peak_kind,
                             statistics.mean(dev_ms), wl.meta["batch"])

    line = {
        "metric": METRIC, "value": value, "unit": "updates/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": tot_dev / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": config_dict(args, wl, world),
        "clocks": clocks,
        "e2e": {"value": e2e_value, "unit": "updates/s", "ms_per_step": tot_e2e / args.steps,
                "h2d_bytes_per_step": int(16 * statistics.mean(len(b) for b in wl.batches[args.warmup:])),
                "d2h_bytes_per_step": int(statsA[-1]["d2h_bytes"]),
                "path": ("bdsm_engine_apply_stream (pinned host buffers, C ABI, host timer around the call)"
                         if pipelined else "bdsm_engine_apply_batch (pinned host buffers, C ABI)")},
        "mode": ("pipelined stream: the timed batches in one bdsm_engine_apply_stream call; the positive phase of "
                 "batch i and the negative phase of batch i+1 share one matching launch (run_pipeline's overlap, "
                 "src/bench.cpp:495-545); ms_per_step = device time of the stream / batches"
                 if pipelined else "one bdsm_engine_apply_batch_device call per batch"),
        "latency": ({"ms_per_batch": statistics.mean(s["ms_device"] for s in statsC),
                     "updates_per_s": updates / (sum(s["ms_device"] for s in statsC) / 1e3),
                     "note": "one batch at a time (bdsm_engine_apply_batch_device), L2 flushed before each, "
                             "validate -> negative -> merge -> positive -> counts",
                     "per_batch_ms": [s["ms_device"] for s in statsC],
                     "neg_ms": [s["ms_negative"] for s in statsC], "merge_ms": [s["ms_update"] for s in statsC],
                     "pos_ms": [s["ms_positive"] for s in statsC]} if statsC else None),
        "gpu_launches": int(sum(s["kernel_launches"] for s in statsA)),
        "cub_launches": int(sum(s["cub_launches"] for s in statsA)),
        "roofline": roof,
        "counts": {"positive": [c for c in flatA[0::2]], "negative": [c for c in flatA[1::2]],
                   "e2e_equals_device_path": parity_ok},
        "per_step": [{"ms": s["ms_device"], "neg_ms": s["ms_negative"], "merge_ms": s["ms_update"],
                      "pos_ms": s["ms_positive"], "match_kernel_ms": s["ms_match_kernel"],
                      "dfs_visits": s["dfs_visits"], "tasks": s["tasks"], "items": s["work_items"],
                      "touched": s["touched"], "relocations": s["relocations"], "attempts": s["attempts"],
                      "reruns": s["reruns"], "compactions": s["compactions"]} for s in statsA],
        "attempts_per_step": [s["attempts"] for s in statsA],
    }
    if world > 1:
        import torch.distributed as dist
        ndev = torch.cuda.device_count()
        line["comm"] = {"backend": dist.get_backend(), "ranks": dist.get_world_size(), "devices": ndev,
                        "step": ("NCCL broadcast of the batch, replicated apply, own share of the work units, "
                                 "NCCL all-reduce of the counts" if dist.get_backend() == "nccl" else
                                 "functional run: ranks share the visible device(s); counts summed over gloo "
                                 "after the timed region")}
    if world == 1 and not args.no_cpu_baseline and wl.meta["E"] > 500_000_000:
        # the reference's PMA alone needs ~69 GB at the
        # Friendster shape plus sort keys and an edge hash set
        line["cpu_baseline"] = {"value": None, "unit": "updates/s", "cores": os.cpu_count(), "kind": "reference",
                                "sample": "not run: the reference's graph build needs > 100 GB of host RAM at "
                                          f"{wl.meta['E']} edges (SURVEY.md §8(d))"}
    tmp = None
    if world == 1 and (args.parity_full != 0 or not args.no_cpu_baseline) and wl.meta["E"] <= 500_000_000:
        tmp = tempfile.mkdtemp(prefix="bdsm_cpu_")
        path = os.path.join(tmp, "workload.bin")
        W.write_file(wl, path)
    if tmp and args.parity_full != 0:
        # Full-scale parity: every batch of the run — warm-up
        # and timed — at full size against the reference-pinned restatement;
        # counts and the reference's dfs_visits must both match.
        nchk = nb if args.parity_full < 0 else min(nb, args.parity_full)
        res = run_restatement_full(path, nchk, args.parity_timeout)
        ours_c = [(flatA[2 * i], flatA[2 * i + 1]) for i in range(nb)]
        ours_v = [None] * args.warmup + [s["dfs_visits"] for s in statsA]
        got = [(b["positive"], b["negative"]) for b in res["batches"]]
        vis = [b["dfs_visits_pruned"] for b in res["batches"]]
        vis_ref = [b["dfs_visits"] for b in res["batches"]]
        eq_counts = got == ours_c[:len(got)]
        # with exact coalescing the engine walks one tree per automorphism orbit,
        # so only the counts are comparable
        eq_vis = None if args.coalesce else all(v is None or v == r for v, r in zip(ours_v, vis))
        line["parity_full"] = {
            "checker": "oracle/oracle_bench: count-only CPU restatement of match_batch (coalesce off), pinned to "
                       "the reference on tests/golden/ (counts, dfs_visits, intersection_ops, tasks_run)",
            "batches": len(got), "batch_updates": wl.meta["batch"], "of": nb, "equal": bool(eq_counts and len(got) == nchk),
            "counts_equal": eq_counts, "dfs_visits_equal": eq_vis,
            "dfs_visits_note": "the engine applies dedupe_by_order at candidate generation, so its dfs_visits is "
                               "the reference tree's minus the subtrees that rule prunes; compared with the "
                               "restatement's count of exactly that tree (dfs_visits_pruned)",
            "reference": got, "ours": ours_c[:len(got)], "dfs_visits_pruned_reference": vis,
            "dfs_visits_reference_tree": vis_ref, "dfs_visits_ours": ours_v[:len(vis)], "cpu_s": res["summary"]["timed_s"] if res["summary"] else None,
            "cores": res["cores"], "max_count": max([max(p) for p in got] or [0])}
    if world == 1 and not args.no_cpu_baseline and tmp:
        res = run_reference_binary(path, args.cpu_prefix, args.cpu_batches, args.cpu_time_cap, timeout=600)
        if res.get("batches"):
            # The reference itself on its feasible sub-batches: replay the same
            # protocol (prefix counted, rest applied) on a fresh engine.
            engC = bd.Engine(wl.labels, wl.src, wl.dst, device=local, chunk=args.chunk)
            engC.add_query(wl.qlabels, wl.qedges)
            ours_sub = []
            for b, ref_b in zip(wl.batches, res["batches"]):
                P = ref_b["updates"]
                r = engC.match_batch(b[:P])
                ours_sub.append((r.positive[0], r.negative[0]))
                if P < len(b):
                    engC.match_batch(b[P:])
            engC.close()
            refc = [(b["positive"], b["negative"]) for b in res["batches"]]
            line["parity_vs_reference"] = {
                "protocol": "reference sub-batches (first P updates of each batch counted, rest applied)",
                "reference": refc, "ours": ours_sub, "equal": refc == ours_sub[:len(refc)]}
        if "summary" in res:
            s = res["summary"]
            line["cpu_baseline"] = {
                "value": s["updates_per_s"], "unit": "updates/s", "cores": res["cores"], "kind": res["kind"],
                "cpu_model": cpu_model(),
                "median_ms_per_subbatch": s["median_ms"],
                "sample": f"first {args.cpu_prefix} updates of each of the first {s['batches']} batches of the "
                          f"same stream (rest applied untimed), {res['cores']} worker threads, "
                          f"coalesce off; graph build {s.get('build_s', 0):.1f}s excluded",
                "per_batch": [{k: b[k] for k in ("positive", "negative", "ms")} for b in res["batches"]]}
        else:
            line["cpu_baseline"] = {"value": None, "unit": "updates/s", "cores": res.get("cores"),
                                    "kind": res.get("kind"), "sample": "failed", "error": res.get("error")}
    if tmp:
        shutil.rmtree(tmp, ignore_errors=True)
    print(json.dumps(line), flush=True)
    engA.close()
    engB.close()
    if engL:
        engL.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())

"""Synthetic workloads for bench.py and the scale tests (BENCH INFRASTRUCTURE).

SURVEY.md §8(d): one seeded generator feeds both the GPU engine and the CPU
baselines (via the binary workload file read by oracle/ref_bench.cpp and
oracle/oracle_bench.cpp), so both consume bit-identical inputs.

  * C1: RMAT (0.57, 0.19, 0.19, 0.05), scale 16, exactly 1M undirected edges,
    8 labels, 4-vertex labelled query, 1K-insert batches.
  * C2: LiveJournal-shaped (4.8M V, 69M E, 16 labels), Chung-Lu power-law
    degrees (max degree capped near LJ's ~2e4, every vertex degree >= 1, ids
    permuted), 6-vertex sparse query, 10K mixed batches.
  * C3/C4/C5 shapes are parameterised the same way.

Sampling semantics follow the reference's generators (src/bench.cpp:67-289):
queries by random-walk extraction with the dense/sparse/tree predicates
(:111-130); batches mixed 2:1 (op = delete iff running index % 3 == 2,
:228-230), inserts uniform over non-edge vertex pairs whose label pair occurs
in G (:233-251), deletes uniform over current edges (:253-266), no pair twice
in a batch, each batch valid against the graph left by the previous one.  The
RNG is torch's (the reference's mt19937 streams are not reproduced; only the
distributions are).  Generation runs on the GPU when one is present.
"""
from __future__ import annotations

import os
import struct
from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np
import torch

NO_LABEL = 0xFFFFFFFF

CONFIGS = {
    "C1": dict(kind="rmat", V=1 << 16, E=1_000_000, L=8, qsize=4, qcat="sparse", batch=1_000,
               mode="insert", desc="Synthetic labelled RMAT 64K vertices / 1M edges, 8 labels, "
                                   "4-vertex labelled query, 1K-edge insert batch"),
    "C2": dict(kind="chunglu", V=4_800_000, E=69_000_000, L=16, qsize=6, qcat="sparse", batch=10_000,
               mode="mixed", dmax=20_000, gamma=2.3,
               desc="LiveJournal-shaped synthetic (4.8M V, 69M E, 16 labels), 6-vertex query, "
                    "10K mixed insert/delete batch"),
    "C3": dict(kind="chunglu", V=3_100_000, E=117_000_000, L=16, qsize=8, qcat="dense", batch=100_000,
               mode="mixed", dmax=33_000, gamma=2.2,
               desc="Orkut-shaped synthetic (3.1M V, 117M E), 8-vertex dense query, 100K-update batch"),
    "C4": dict(kind="chunglu_lean", V=65_000_000, E=1_800_000_000, L=16, qsize=6, qcat="sparse",
               batch=1_000_000, mode="mixed", dmax=5_214, gamma=2.5,
               desc="Friendster-shaped synthetic (65M V, 1.8B E, 16 labels), 6-vertex query, 1M-update batch"),
    "C5": dict(kind="chunglu", V=1_000_000, E=10_000_000, L=1, qsize=5, qcat="clique", batch=10_000,
               mode="mixed", dmax=5_000, gamma=2.3,
               desc="Batch-size sweep with unlabelled 5-vertex clique query"),
    "C5cycle": dict(kind="chunglu", V=1_000_000, E=10_000_000, L=1, qsize=5, qcat="cycle", batch=10_000,
                    mode="mixed", dmax=5_000, gamma=2.3,
                    desc="Batch-size sweep with unlabelled 5-cycle query"),
}


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return g


def _dedupe_first(u: torch.Tensor, v: torch.Tensor, want: int) -> Tuple[torch.Tensor, torch.Tensor, int]:
    """Drops self-loops and repeated pairs (keeping the first occurrence in
    generation order) and returns the first `want` survivors."""
    keep = u != v
    u, v = u[keep], v[keep]
    a, b = torch.minimum(u, v), torch.maximum(u, v)
    key = (a << 32) | b
    skey, order = torch.sort(key, stable=True)
    first = torch.ones_like(skey, dtype=torch.bool)
    first[1:] = skey[1:] != skey[:-1]
    idx = torch.sort(order[first]).values
    got = int(idx.numel())
    idx = idx[:want]
    return a[idx], b[idx], got


def rmat_graph(scale: int, E: int, seed: int, device, probs=(0.57, 0.19, 0.19, 0.05)):
    g = _gen(seed, device)
    V = 1 << scale
    cum = torch.tensor(np.cumsum(probs)[:3], dtype=torch.float32, device=device)
    us, vs = [], []
    have = 0
    mult = 1.3
    while True:
        n = int(E * mult) + 1024
        u = torch.zeros(n, dtype=torch.int64, device=device)
        v = torch.zeros(n, dtype=torch.int64, device=device)
        for bit in range(scale):
            r = torch.rand(n, generator=g, device=device)
            q = torch.bucketize(r, cum)  # 0..3 quadrant
            u |= ((q >> 1) & 1) << bit
            v |= (q & 1) << bit
        us.append(u)
        vs.append(v)
        a, b, got = _dedupe_first(torch.cat(us), torch.cat(vs), E)
        if got >= E:
            return V, a, b
        mult *= 1.5


def _host_cdf(V: int, E: int, dmax: int, gamma: float) -> np.ndarray:
    """Chung-Lu endpoint CDF: power-law expected degrees w_i ~ (i+1)^(-1/(gamma-1)),
    scaled to mean 2E/V under the cap dmax; float64 on the host (sequential sums)."""
    alpha = 1.0 / (gamma - 1.0)
    w = (np.arange(V, dtype=np.float64) + 1.0) ** (-alpha)
    target = 2.0 * E / V
    for _ in range(50):  # scale to the mean degree under the cap
        w = w * (target * V / float(w.sum()))
        w = np.minimum(w, float(dmax))
        if abs(float(w.sum()) / V - target) < 1e-3 * target:
            break
    cdf = np.cumsum(w)
    return cdf / cdf[-1]


def chung_lu_graph(V: int, E: int, seed: int, device, dmax: int, gamma: float):
    """Power-law expected degrees w_i ~ (i+i0)^(-1/(gamma-1)), mean 2E/V, capped
    at dmax; one guaranteed edge per vertex (no isolated vertices), the rest
    sampled with both endpoints proportional to w; ids randomly permuted."""
    g = _gen(seed, device)
    # weights and CDF on the host: numpy's sequential float64 sums are
    # reproducible across devices and boxes, a device scan's association
    # order is not (and the CDF decides every endpoint draw)
    cdf = torch.from_numpy(_host_cdf(V, E, dmax, gamma)).to(device)
    perm = torch.randperm(V, generator=g, device=device)

    def draw(n):
        r = torch.rand(n, generator=g, device=device, dtype=torch.float64)
        return torch.clamp(torch.searchsorted(cdf, r), max=V - 1)

    base_u = torch.arange(V, device=device)
    base_v = draw(V)
    base_v = torch.where(base_v == base_u, (base_v + 1) % V, base_v)
    us, vs = [base_u], [base_v]
    mult = 1.05
    while True:
        n = int((E - V) * mult) + 4096
        us.append(draw(n))
        vs.append(draw(n))
        a, b, got = _dedupe_first(torch.cat(us), torch.cat(vs), E)
        if got >= E:
            break
        mult = 0.2 * (E - got) / max(E, 1) + 0.02
    a, b = perm[a], perm[b]
    return V, torch.minimum(a, b), torch.maximum(a, b)


def chung_lu_keys(V: int, E: int, seed: int, device, dmax: int, gamma: float, chunk: int = 1 << 27):
    """Memory-lean Chung-Lu for billion-edge shapes (C4): the same weight
    sequence and one guaranteed edge per vertex as chung_lu_graph, sampled in
    chunks straight into undirected keys (min << 32 | max); duplicates and
    self-loops dropped, topped up until >= E, then a uniformly random surplus
    removed, so exactly E edges.  Returns the sorted int64 keys (one array of
    8 B per edge instead of the per-step copies of the small-shape path)."""
    g = _gen(seed, device)
    cdf = torch.from_numpy(_host_cdf(V, E, dmax, gamma)).to(device)
    perm = torch.randperm(V, generator=g, device=device)

    def keys_of(u, v):
        u, v = perm[u], perm[v]
        keep = u != v
        u, v = u[keep], v[keep]
        return (torch.minimum(u, v) << 32) | torch.maximum(u, v)

    def draw(n):
        r = torch.rand(n, generator=g, device=device, dtype=torch.float64)
        return torch.clamp(torch.searchsorted(cdf, r), max=V - 1)

    base_u = torch.arange(V, device=device)
    base_v = draw(V)
    base_v = torch.where(base_v == base_u, (base_v + 1) % V, base_v)
    parts = [keys_of(base_u, base_v)]
    del base_u, base_v
    want = int((E - V) * 1.03) + 4096
    while want > 0:
        c = min(chunk, want)
        parts.append(keys_of(draw(c), draw(c)))
        want -= c
    keys = torch.unique(torch.cat(parts))
    del parts
    while keys.numel() < E:  # top up
        more = []
        need = int((E - keys.numel()) * 1.5) + 4096
        while need > 0:
            c = min(chunk, need)
            more.append(keys_of(draw(c), draw(c)))
            need -= c
        extra = torch.unique(torch.cat(more))
        pos = torch.clamp(torch.searchsorted(keys, extra), max=keys.numel() - 1)
        extra = extra[keys[pos] != extra]
        keys = torch.sort(torch.cat([keys, extra])).values
    surplus = keys.numel() - E
    if surplus > 0:  # drop a uniformly random surplus
        drop = torch.empty(0, dtype=torch.int64, device=device)
        while drop.numel() < surplus:
            drop = torch.unique(torch.cat([drop, torch.randint(0, keys.numel(), (2 * surplus + 16,), generator=g,
                                                               device=device)]))
        drop = drop[torch.randperm(drop.numel(), generator=g, device=device)[:surplus]]
        keep = torch.ones(keys.numel(), dtype=torch.bool, device=device)
        keep[drop] = False
        keys = keys[keep]
    return V, keys


class _KeysGraph:
    """Neighbour queries and degrees straight from the sorted undirected keys
    (billion-edge shapes, where the directed CSR copy would not fit)."""

    def __init__(self, keys: torch.Tensor, V: int):
        self.keys = keys
        self.V = V
        # the reverse direction (max << 32 | min), sorted, so a neighbour query is two range lookups
        self.rkeys = torch.sort(((keys & 0xFFFFFFFF) << 32) | (keys >> 32)).values
        deg = torch.zeros(V, dtype=torch.int64, device=keys.device)
        step = 1 << 28
        for s in range(0, keys.numel(), step):
            k = keys[s:s + step]
            deg += torch.bincount(k >> 32, minlength=V) + torch.bincount(k & 0xFFFFFFFF, minlength=V)
        self.deg = deg
        self.off_h = None

    def degree(self, u: int) -> int:
        return int(self.deg[u])

    def neighbors(self, u: int) -> np.ndarray:
        bounds = torch.tensor([u << 32, (u + 1) << 32], device=self.keys.device)
        lo, hi = torch.searchsorted(self.keys, bounds).tolist()
        rlo, rhi = torch.searchsorted(self.rkeys, bounds).tolist()
        both = torch.cat([self.keys[lo:hi], self.rkeys[rlo:rhi]]) & 0xFFFFFFFF
        return torch.sort(both).values.cpu().numpy()


@dataclass
class Workload:
    name: str
    V: int
    labels: np.ndarray          # u32 [V]
    src: np.ndarray             # u32 [E]
    dst: np.ndarray
    qlabels: List[int]
    qedges: List[Tuple[int, int]]
    batches: List[np.ndarray]   # structured UPDATE arrays (u, v, op, elab)
    meta: dict = field(default_factory=dict)


UPDATE_DTYPE = np.dtype([("u", "<u4"), ("v", "<u4"), ("op", "<u4"), ("elab", "<u4")])


class _HostCSR:
    """Sorted directed keys on the generation device for neighbour queries."""

    def __init__(self, a: torch.Tensor, b: torch.Tensor, V: int):
        keys = torch.cat([(a << 32) | b, (b << 32) | a])
        self.keys = torch.sort(keys).values
        src = self.keys >> 32
        counts = torch.bincount(src, minlength=V)
        self.off = torch.zeros(V + 1, dtype=torch.int64, device=a.device)
        self.off[1:] = torch.cumsum(counts, 0)
        self.deg = counts
        self.off_h = self.off.cpu().numpy()

    def degree(self, u: int) -> int:
        return int(self.off_h[u + 1] - self.off_h[u])

    def neighbors(self, u: int) -> np.ndarray:
        lo, hi = int(self.off_h[u]), int(self.off_h[u + 1])
        return (self.keys[lo:hi] & 0xFFFFFFFF).cpu().numpy()


def extract_query(csr: _HostCSR, labels: np.ndarray, size: int, category: str, seed: int,
                  attempts: int = 4000):
    """Random-walk query extraction with the reference's predicates
    (src/bench.cpp:67-140)."""
    rng = np.random.default_rng(seed)
    V = len(labels)
    for _ in range(attempts):
        start = int(rng.integers(0, V))
        if csr.degree(start) == 0:
            continue
        members = [start]
        mset = {start}
        tree = []
        stuck = 0
        cache = {}
        while len(members) < size and stuck < 64 * size:
            u = members[int(rng.integers(0, len(members)))]
            nb = cache.get(u)
            if nb is None:
                nb = cache[u] = csr.neighbors(u)
            if len(nb) == 0:
                stuck += 1
                continue
            w = int(nb[int(rng.integers(0, len(nb)))])
            if w in mset:
                stuck += 1
                continue
            members.append(w)
            mset.add(w)
            tree.append((u, w))
            stuck = 0
        if len(members) < size:
            continue
        members.sort()
        local = {m: i for i, m in enumerate(members)}
        if category == "tree":
            edges = [(local[u], local[w]) for u, w in tree]
        else:
            edges = []
            for u in members:
                nb = cache.get(u)
                if nb is None:
                    nb = cache[u] = csr.neighbors(u)
                for w in nb:
                    w = int(w)
                    if w > u and w in mset:
                        edges.append((local[u], local[w]))
            d_avg = 2.0 * len(edges) / size
            if category == "dense" and d_avg < 3.0:
                continue
            if category == "sparse" and (d_avg >= 3.0 or len(edges) < size):
                continue
        return [int(labels[m]) for m in members], edges
    raise RuntimeError(f"could not extract a {category} query of size {size}")


def make_stream(a: Optional[torch.Tensor], b: Optional[torch.Tensor], labels_t: torch.Tensor, V: int,
                nbatches: int, batch: int, mode: str, seed: int,
                keys: Optional[torch.Tensor] = None) -> List[np.ndarray]:
    """Mixed/insert/delete batches with the reference's sampling semantics
    (src/bench.cpp:222-287), vectorised: candidates are drawn in bulk and the
    first valid ones in draw order are taken.  `keys` (sorted undirected
    min << 32 | max) replaces a, b for billion-edge shapes."""
    device = labels_t.device
    g = _gen(seed, device)
    if keys is None:
        keys = torch.sort((a << 32) | b).values  # current undirected edge set, sorted
    L = int(labels_t.max()) + 1
    lp = torch.zeros(L * L, dtype=torch.bool, device=device)
    step = 1 << 28
    for s0 in range(0, keys.numel(), step):  # label pairs present in G
        k = keys[s0:s0 + step]
        la, lb = labels_t[k >> 32], labels_t[k & 0xFFFFFFFF]
        lp[torch.minimum(la, lb) * L + torch.maximum(la, lb)] = True
        del la, lb
    out = []
    emitted = 0
    for _ in range(nbatches):
        ops = np.zeros(batch, np.uint32)
        if mode == "mixed":
            ops = (((np.arange(batch) + emitted) % 3) == 2).astype(np.uint32)
        elif mode == "delete":
            ops[:] = 1
        n_del = int(ops.sum())
        n_ins = batch - n_del
        # inserts: uniform u != v, non-edge, label pair present, not repeated
        ins_u = torch.empty(0, dtype=torch.int64, device=device)
        ins_v = torch.empty(0, dtype=torch.int64, device=device)
        while ins_u.numel() < n_ins:
            n = 2 * (n_ins - ins_u.numel()) + 1024
            u = torch.randint(0, V, (n,), generator=g, device=device)
            v = torch.randint(0, V, (n,), generator=g, device=device)
            mn, mx = torch.minimum(u, v), torch.maximum(u, v)
            k = (mn << 32) | mx
            ok = u != v
            pos = torch.searchsorted(keys, k)
            pos = torch.clamp(pos, max=keys.numel() - 1)
            ok &= keys[pos] != k
            lu, lv = labels_t[u], labels_t[v]
            ok &= lp[torch.minimum(lu, lv) * L + torch.maximum(lu, lv)]
            u, v = u[ok], v[ok]
            cu = torch.cat([ins_u, u])
            cv = torch.cat([ins_v, v])
            # first occurrence of each pair in draw order, drawn orientation kept
            ck = (torch.minimum(cu, cv) << 32) | torch.maximum(cu, cv)
            sk, order = torch.sort(ck, stable=True)
            first = torch.ones_like(sk, dtype=torch.bool)
            first[1:] = sk[1:] != sk[:-1]
            idx = torch.sort(order[first]).values[:n_ins]
            ins_u, ins_v = cu[idx], cv[idx]
        # deletes: uniform over current edges, not repeated
        del_idx = torch.empty(0, dtype=torch.int64, device=device)
        while del_idx.numel() < n_del:
            n = 2 * (n_del - del_idx.numel()) + 1024
            r = torch.randint(0, keys.numel(), (n,), generator=g, device=device)
            c = torch.cat([del_idx, r])
            sk, order = torch.sort(c, stable=True)
            first = torch.ones_like(sk, dtype=torch.bool)
            first[1:] = sk[1:] != sk[:-1]
            del_idx = c[torch.sort(order[first]).values][:n_del]
        dk = keys[del_idx]
        arr = np.zeros(batch, dtype=UPDATE_DTYPE)
        ins_pos = np.nonzero(ops == 0)[0]
        del_pos = np.nonzero(ops == 1)[0]
        arr["u"][ins_pos] = ins_u.cpu().numpy().astype(np.uint32)
        arr["v"][ins_pos] = ins_v.cpu().numpy().astype(np.uint32)
        dkh = dk.cpu().numpy()
        arr["u"][del_pos] = (dkh >> 32).astype(np.uint32)
        arr["v"][del_pos] = (dkh & 0xFFFFFFFF).astype(np.uint32)
        arr["op"] = ops
        arr["elab"] = NO_LABEL
        out.append(arr)
        emitted += batch
        # advance the edge set
        keep = torch.ones(keys.numel(), dtype=torch.bool, device=device)
        keep[del_idx] = False
        ik = (torch.minimum(ins_u, ins_v) << 32) | torch.maximum(ins_u, ins_v)
        keys = torch.sort(torch.cat([keys[keep], ik])).values
    return out


def build(name: str, nbatches: int, seed_graph: int = 1, seed_query: int = 7, seed_stream: int = 9,
          device=None, batch: Optional[int] = None, scale_down: int = 1) -> Workload:
    """Generates config `name` ("C1", "C2", ...).  scale_down > 1 shrinks V and
    E proportionally (tests)."""
    cfg = dict(CONFIGS[name])
    if device is None:
        device = "cuda" if torch.cuda.is_available() else "cpu"
    V, E = cfg["V"] // scale_down, cfg["E"] // scale_down
    keys = None
    if cfg["kind"] == "rmat":
        scale = max(4, int(np.log2(V)))
        V, a, b = rmat_graph(scale, E, seed_graph, device)
    elif cfg["kind"] == "chunglu_lean":
        V, keys = chung_lu_keys(V, E, seed_graph, device, max(16, cfg["dmax"] // scale_down), cfg["gamma"])
        a = b = None
    else:
        V, a, b = chung_lu_graph(V, E, seed_graph, device, max(16, cfg["dmax"] // scale_down), cfg["gamma"])
    lg = _gen(seed_graph + 1, device)
    labels_t = torch.randint(0, cfg["L"], (V,), generator=lg, device=device)
    csr = _HostCSR(a, b, V) if keys is None else _KeysGraph(keys, V)
    labels = labels_t.cpu().numpy().astype(np.uint32)
    if cfg["qcat"] == "clique":
        n = cfg["qsize"]
        ql = [0] * n
        qe = [(i, j) for i in range(n) for j in range(i + 1, n)]
    elif cfg["qcat"] == "cycle":
        n = cfg["qsize"]
        ql = [0] * n
        qe = [(i, (i + 1) % n) for i in range(n)]
    else:
        # sparse queries need an induced cycle, rare in a walk over a 1.8B-edge
        # graph with mean degree 55: more attempts for the billion-edge shape
        ql, qe = extract_query(csr, labels, cfg["qsize"], cfg["qcat"], seed_query,
                               attempts=40000 if keys is not None else 4000)
    bsz = batch or cfg["batch"]
    batches = make_stream(a, b, labels_t, V, nbatches, bsz, cfg["mode"], seed_stream, keys=keys)
    deg = csr.deg
    meta = {"V": V, "E": int(a.numel()) if keys is None else int(keys.numel()), "L": cfg["L"], "d_max": int(deg.max()), "d_mean": float(deg.float().mean()),
            "isolated": int((deg == 0).sum()), "batch": bsz, "mode": cfg["mode"], "generator": cfg["kind"],
            "seeds": {"graph": seed_graph, "query": seed_query, "stream": seed_stream}, "desc": cfg["desc"]}
    if keys is not None:  # u32 endpoint arrays, converted in slices
        del csr.rkeys
        src = np.empty(keys.numel(), np.uint32)
        dst = np.empty(keys.numel(), np.uint32)
        step = 1 << 28
        for s0 in range(0, keys.numel(), step):
            k = keys[s0:s0 + step]
            src[s0:s0 + k.numel()] = (k >> 32).to(torch.int32).cpu().numpy().view(np.uint32)
            dst[s0:s0 + k.numel()] = (k & 0xFFFFFFFF).to(torch.int32).cpu().numpy().view(np.uint32)
        del keys
    else:
        src, dst = a.cpu().numpy().astype(np.uint32), b.cpu().numpy().astype(np.uint32)
    wl = Workload(name, V, labels, src, dst, ql, qe, batches, meta)
    del csr
    if torch.cuda.is_available():
        torch.cuda.empty_cache()
    return wl


def write_file(wl: Workload, path: str, nbatches: Optional[int] = None) -> None:
    """Binary workload file (layout in oracle/workload.hpp)."""
    bs = wl.batches if nbatches is None else wl.batches[:nbatches]
    total = sum(len(b) for b in bs)
    with open(path, "wb") as f:
        f.write(b"BDSMWL01")
        f.write(struct.pack("<7Q", wl.V, len(wl.src), 0, len(wl.qlabels), len(wl.qedges), len(bs), total))
        f.write(np.asarray(wl.labels, np.uint32).tobytes())
        f.write(np.asarray(wl.src, np.uint32).tobytes())
        f.write(np.asarray(wl.dst, np.uint32).tobytes())
        f.write(np.asarray(wl.qlabels, np.uint32).tobytes())
        f.write(np.asarray([e[0] for e in wl.qedges], np.uint32).tobytes())
        f.write(np.asarray([e[1] for e in wl.qedges], np.uint32).tobytes())
        f.write(np.full(len(wl.qedges), NO_LABEL, np.uint32).tobytes())
        offs = np.cumsum([0] + [len(b) for b in bs]).astype(np.uint64)
        f.write(offs.tobytes())
        cat = np.concatenate(bs) if bs else np.zeros(0, UPDATE_DTYPE)
        for fld in ("u", "v", "op", "elab"):
            f.write(np.ascontiguousarray(cat[fld]).astype(np.uint32).tobytes())

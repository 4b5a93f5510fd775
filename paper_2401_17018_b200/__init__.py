"""B200-native batch-dynamic subgraph matching (GAMMA, arXiv 2401.17018).

Python binding of the C ABI in include/bdsm_gpu.h (libbdsm_b200.so, built
in-tree by paper_2401_17018_b200/build.sh).  It mirrors the reference's
bdsm_core API for the hot path:

  reference (C++)                                  here
  ----------------------------------------------   -----------------------------
  LabeledGraph::build_from_edges (graph.cpp:35)    Engine(vlabels, src, dst, ...)
  QueryGraph + QueryEncodingState::initialize +
    build_query_plan (coalesce off)                Engine.add_query(labels, edges)
  UpdateBatch + match_batch (matcher.cpp:370)      Engine.match_batch(updates)
  BatchError / std::invalid_argument               BatchError / ValueError

The engine returns per-query counts |positive| and |negative| (the reference
returns the match vectors whose sizes the CLI reports in deltas.csv).  There
is no CPU fallback: importing this package without the built library raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Iterable, List, Optional, Sequence, Tuple

import numpy as np

__all__ = ["Engine", "BatchError", "EngineError", "UPDATE_DTYPE", "make_updates", "lib_path",
           "shard_owners", "NO_LABEL"]

NO_LABEL = 0xFFFFFFFF
_HERE = os.path.dirname(os.path.abspath(__file__))


def lib_path() -> str:
    # BDSM_LIB: an alternative build of the same engine (e.g. -DBDSM_TRACE diagnostics)
    return os.environ.get("BDSM_LIB") or os.path.join(_HERE, "libbdsm_b200.so")


UPDATE_DTYPE = np.dtype([("u", "<u4"), ("v", "<u4"), ("op", "<u4"), ("elab", "<u4")])


class _GraphDesc(C.Structure):
    _fields_ = [("num_vertices", C.c_uint32), ("vertex_labels", C.c_void_p), ("num_edges", C.c_uint64),
                ("src", C.c_void_p), ("dst", C.c_void_p), ("edge_labels", C.c_void_p)]


class _QueryDesc(C.Structure):
    _fields_ = [("num_vertices", C.c_uint32), ("vertex_labels", C.c_void_p), ("num_edges", C.c_uint32),
                ("a", C.c_void_p), ("b", C.c_void_p), ("edge_labels", C.c_void_p)]


class _Options(C.Structure):
    _fields_ = [("group_bits", C.c_uint32), ("coalesce", C.c_uint32), ("device", C.c_int32),
                ("shard_rank", C.c_uint32), ("shard_world", C.c_uint32), ("slack", C.c_float),
                ("pool_reserve", C.c_float), ("chunk", C.c_uint32), ("zero_copy", C.c_uint32),
                ("l2_hot_mb", C.c_uint32)]


class _UpdateError(C.Structure):
    _fields_ = [("index", C.c_uint64), ("reason", C.c_uint32)]


class _Stats(C.Structure):
    _fields_ = [("ms_total", C.c_double), ("ms_device", C.c_double), ("ms_negative", C.c_double),
                ("ms_update", C.c_double), ("ms_positive", C.c_double), ("dfs_visits", C.c_uint64),
                ("tasks", C.c_uint64), ("work_items", C.c_uint64), ("gen_calls", C.c_uint64),
                ("bytes_phase", C.c_uint64), ("bytes_update", C.c_uint64), ("touched", C.c_uint64),
                ("relocations", C.c_uint64), ("compactions", C.c_uint32), ("timed_out", C.c_uint32),
                ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64), ("ms_match_kernel", C.c_double),
                ("ms_merge_kernel", C.c_double), ("kernel_launches", C.c_uint32), ("cub_launches", C.c_uint32),
                ("bytes_kernel", C.c_uint64), ("attempts", C.c_uint32), ("reruns", C.c_uint32)]


_lib = None


def _load():
    global _lib
    if _lib is not None:
        return _lib
    path = lib_path()
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build the CUDA engine first "
            "(python -c 'import __graft_entry__ as g; g.build()' or paper_2401_17018_b200/build.sh)")
    L = C.CDLL(path)
    L.bdsm_engine_create.restype = C.c_int
    L.bdsm_engine_create.argtypes = [C.POINTER(_GraphDesc), C.POINTER(_Options), C.POINTER(C.c_void_p)]
    L.bdsm_engine_destroy.restype = None
    L.bdsm_engine_destroy.argtypes = [C.c_void_p]
    L.bdsm_engine_add_query.restype = C.c_int
    L.bdsm_engine_add_query.argtypes = [C.c_void_p, C.POINTER(_QueryDesc)]
    for name in ("bdsm_engine_apply_batch", "bdsm_engine_apply_batch_device"):
        f = getattr(L, name)
        f.restype = C.c_int
        f.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p, C.POINTER(_Stats)]
    L.bdsm_engine_submit_batch.restype = C.c_int
    L.bdsm_engine_submit_batch.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t]
    L.bdsm_engine_wait.restype = C.c_int
    L.bdsm_engine_wait.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(_Stats)]
    L.bdsm_engine_set_deadline.restype = C.c_int
    L.bdsm_engine_set_deadline.argtypes = [C.c_void_p, C.c_int, C.c_double]
    L.bdsm_engine_apply_stream.restype = C.c_int
    L.bdsm_engine_apply_stream.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p,
                                           C.c_void_p, C.c_void_p, C.c_void_p]
    L.bdsm_engine_set_query_active.restype = C.c_int
    L.bdsm_engine_set_query_active.argtypes = [C.c_void_p, C.c_int, C.c_int]
    L.bdsm_engine_query_timed_out.restype = C.c_int
    L.bdsm_engine_query_timed_out.argtypes = [C.c_void_p, C.c_int]
    L.bdsm_last_batch_errors.restype = C.c_size_t
    L.bdsm_last_batch_errors.argtypes = [C.c_void_p, C.POINTER(_UpdateError), C.c_size_t]
    L.bdsm_last_error.restype = C.c_char_p
    L.bdsm_last_error.argtypes = []
    L.bdsm_engine_neighbors.restype = C.c_size_t
    L.bdsm_engine_neighbors.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p, C.c_size_t]
    L.bdsm_engine_rows.restype = C.c_int
    L.bdsm_engine_rows.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
    L.bdsm_engine_order.restype = C.c_int
    L.bdsm_engine_order.argtypes = [C.c_void_p, C.c_int, C.c_uint32, C.c_void_p]
    L.bdsm_engine_column_sizes.restype = C.c_int
    L.bdsm_engine_column_sizes.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
    L.bdsm_engine_replan.restype = C.c_int
    L.bdsm_engine_replan.argtypes = [C.c_void_p, C.c_int]
    L.bdsm_engine_num_edges.restype = C.c_uint64
    L.bdsm_engine_num_edges.argtypes = [C.c_void_p]
    L.bdsm_engine_num_vertices.restype = C.c_uint32
    L.bdsm_engine_num_vertices.argtypes = [C.c_void_p]
    L.bdsm_shard_owners.restype = None
    L.bdsm_shard_owners.argtypes = [C.c_void_p, C.c_size_t, C.c_uint32, C.c_void_p]
    L.bdsm_engine_debug_trace.restype = C.c_size_t
    L.bdsm_engine_debug_trace.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t]
    L.bdsm_engine_collect_matches.restype = C.c_int
    L.bdsm_engine_collect_matches.argtypes = [C.c_void_p, C.c_uint64]
    L.bdsm_engine_matches.restype = C.c_int64
    L.bdsm_engine_matches.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_size_t]
    L.bdsm_engine_tail.restype = C.c_int
    L.bdsm_engine_tail.argtypes = [C.c_void_p, C.c_int, C.c_uint32]
    L.bdsm_plan_edge_orbits.restype = C.c_int64
    L.bdsm_plan_edge_orbits.argtypes = [C.c_void_p, C.c_void_p]
    L.bdsm_version.restype = C.c_char_p
    L.bdsm_version.argtypes = []
    # multi-device engine group (bdsm_group_*)
    L.bdsm_group_create.restype = C.c_int
    L.bdsm_group_create.argtypes = [C.POINTER(_GraphDesc), C.POINTER(_Options), C.c_void_p, C.c_uint32,
                                    C.POINTER(C.c_void_p)]
    L.bdsm_group_destroy.restype = None
    L.bdsm_group_destroy.argtypes = [C.c_void_p]
    L.bdsm_group_size.restype = C.c_uint32
    L.bdsm_group_size.argtypes = [C.c_void_p]
    L.bdsm_group_engine.restype = C.c_void_p
    L.bdsm_group_engine.argtypes = [C.c_void_p, C.c_uint32]
    L.bdsm_group_add_query.restype = C.c_int
    L.bdsm_group_add_query.argtypes = [C.c_void_p, C.POINTER(_QueryDesc)]
    L.bdsm_group_apply_batch.restype = C.c_int
    L.bdsm_group_apply_batch.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p,
                                         C.POINTER(_Stats)]
    L.bdsm_group_submit_batch.restype = C.c_int
    L.bdsm_group_submit_batch.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t]
    L.bdsm_group_wait.restype = C.c_int
    L.bdsm_group_wait.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(_Stats)]
    L.bdsm_group_apply_stream.restype = C.c_int
    L.bdsm_group_apply_stream.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p,
                                          C.c_void_p, C.c_void_p]
    L.bdsm_group_set_query_active.restype = C.c_int
    L.bdsm_group_set_query_active.argtypes = [C.c_void_p, C.c_int, C.c_int]
    L.bdsm_group_collect_matches.restype = C.c_int
    L.bdsm_group_collect_matches.argtypes = [C.c_void_p, C.c_uint64]
    L.bdsm_group_matches.restype = C.c_int64
    L.bdsm_group_matches.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_size_t]
    _lib = L
    return L


def lib():
    return _load()


class EngineError(RuntimeError):
    """Non-batch failure (CUDA error, out of memory, runtime error)."""

    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


class BatchError(RuntimeError):
    """bdsm::BatchError (include/bdsm/graph.hpp:42-52): all-or-nothing rejection.
    failures: list of (index, reason) with reason 1 unknown vertex, 2 insert of
    an existing edge, 3 delete of a missing edge."""

    def __init__(self, msg: str, failures):
        super().__init__(msg)
        self.failures = failures


_REASONS = {1: "unknown vertex", 2: "insert of existing edge", 3: "delete of missing edge"}


def _raise(status: int, engine_handle=None):
    msg = (lib().bdsm_last_error() or b"").decode()
    if status == 1:
        fails = []
        if engine_handle:
            n = lib().bdsm_last_batch_errors(engine_handle, None, 0)
            buf = (_UpdateError * max(n, 1))()
            lib().bdsm_last_batch_errors(engine_handle, buf, n)
            fails = [(int(buf[i].index), int(buf[i].reason)) for i in range(n)]
        raise BatchError(msg, fails)
    if status == 2:
        raise ValueError(msg)
    if status == 5:
        raise MemoryError(msg)
    raise EngineError(status, msg)


def _u32(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.uint32))


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else C.c_void_p(a.ctypes.data)


def make_updates(updates) -> np.ndarray:
    """Packs updates into the C ABI layout (bdsm_update: u, v, op, edge_label).
    Accepts a structured array of UPDATE_DTYPE, an (n, 3|4) integer array, or an
    iterable of (op, u, v[, label]) tuples with op 0 insert / 1 delete (the
    tests' tuple order)."""
    if isinstance(updates, np.ndarray) and updates.dtype == UPDATE_DTYPE:
        return np.ascontiguousarray(updates)
    rows = list(updates)
    out = np.zeros(len(rows), dtype=UPDATE_DTYPE)
    for i, r in enumerate(rows):
        op, u, v = int(r[0]), int(r[1]), int(r[2])
        lab = r[3] if len(r) > 3 else None
        out[i] = (u, v, op, NO_LABEL if lab is None or lab < 0 else lab)
    return out


@dataclass
class BatchResult:
    positive: List[int]
    negative: List[int]
    stats: dict = field(default_factory=dict)


def _stats_dict(s: _Stats) -> dict:
    return {name: getattr(s, name) for name, _ in _Stats._fields_}


class Engine:
    """Device-resident dynamic graph + registered queries (one CUDA device)."""

    def __init__(self, vertex_labels, src, dst, edge_labels=None, *, group_bits: int = 2, device: int = 0,
                 shard_rank: int = 0, shard_world: int = 1, slack: float = 0.25, pool_reserve: float = 0.5,
                 chunk: int = 32, zero_copy: bool = False, l2_hot_mb: int = 0, coalesce: bool = False):
        L = lib()
        self._vl = _u32(vertex_labels)
        s, d = _u32(src), _u32(dst)
        el = None if edge_labels is None else _u32(edge_labels)
        desc = _GraphDesc(len(self._vl), self._vl.ctypes.data, len(s), s.ctypes.data, d.ctypes.data,
                          None if el is None else el.ctypes.data)
        opts = _Options(group_bits, 1 if coalesce else 0, device, shard_rank, shard_world, slack, pool_reserve, chunk,
                        1 if zero_copy else 0, l2_hot_mb)
        h = C.c_void_p()
        st = L.bdsm_engine_create(C.byref(desc), C.byref(opts), C.byref(h))
        if st != 0:
            _raise(st)
        self._h = h
        self.nq = 0
        self.query_sizes: List[int] = []

    @property
    def handle(self):
        return self._h

    def add_query(self, labels: Sequence[int], edges: Iterable[Tuple]) -> int:
        ql = _u32(labels)
        edges = list(edges)
        qa = _u32([e[0] for e in edges])
        qb = _u32([e[1] for e in edges])
        qlab = _u32([NO_LABEL if (len(e) < 3 or e[2] is None or e[2] < 0) else e[2] for e in edges])
        desc = _QueryDesc(len(ql), ql.ctypes.data, len(qa), qa.ctypes.data if len(qa) else None,
                          qb.ctypes.data if len(qb) else None, qlab.ctypes.data if len(qlab) else None)
        r = lib().bdsm_engine_add_query(self._h, C.byref(desc))
        if r < 0:
            _raise(-r, self._h)
        self.nq += 1
        self.query_sizes.append(len(ql))
        return r

    def match_batch(self, updates) -> BatchResult:
        """match_batch over every query; updates in HOST memory."""
        ups = make_updates(updates)
        pos = np.zeros(max(self.nq, 1), np.uint64)
        neg = np.zeros(max(self.nq, 1), np.uint64)
        st = _Stats()
        r = lib().bdsm_engine_apply_batch(self._h, _ptr(ups) if len(ups) else None, len(ups), _ptr(pos),
                                          _ptr(neg), C.byref(st))
        if r != 0:
            _raise(r, self._h)
        return BatchResult(pos[: self.nq].tolist(), neg[: self.nq].tolist(), _stats_dict(st))

    apply_batch = match_batch

    def submit_batch(self, updates) -> None:
        """Pipelined match_batch, first half: stages the host batch and
        enqueues it; returns at once (the caller may reuse `updates`)."""
        ups = make_updates(updates)
        r = lib().bdsm_engine_submit_batch(self._h, _ptr(ups) if len(ups) else None, len(ups))
        if r != 0:
            _raise(r, self._h)

    def wait(self) -> BatchResult:
        """Second half: the submitted batch's result (as match_batch)."""
        pos = np.zeros(max(self.nq, 1), np.uint64)
        neg = np.zeros(max(self.nq, 1), np.uint64)
        st = _Stats()
        r = lib().bdsm_engine_wait(self._h, _ptr(pos), _ptr(neg), C.byref(st))
        if r != 0:
            _raise(r, self._h)
        return BatchResult(pos[: self.nq].tolist(), neg[: self.nq].tolist(), _stats_dict(st))

    def match_batch_device(self, dev_ptr: int, n: int) -> BatchResult:
        """Same, with the packed updates already in device memory (e.g. a
        torch uint8/int32 CUDA tensor's data_ptr())."""
        pos = np.zeros(max(self.nq, 1), np.uint64)
        neg = np.zeros(max(self.nq, 1), np.uint64)
        st = _Stats()
        r = lib().bdsm_engine_apply_batch_device(self._h, C.c_void_p(dev_ptr), n, _ptr(pos), _ptr(neg),
                                                 C.byref(st))
        if r != 0:
            _raise(r, self._h)
        return BatchResult(pos[: self.nq].tolist(), neg[: self.nq].tolist(), _stats_dict(st))

    def _stream(self, ptrs, sizes, device: bool) -> List[BatchResult]:
        k, nq = len(sizes), max(self.nq, 1)
        parr = (C.c_void_p * max(k, 1))(*[C.c_void_p(int(x)) for x in ptrs])
        sarr = (C.c_size_t * max(k, 1))(*[int(s) for s in sizes])
        pos = np.zeros(max(k * nq, 1), np.uint64)
        neg = np.zeros(max(k * nq, 1), np.uint64)
        stats = (_Stats * max(k, 1))()
        done = C.c_size_t(0)
        r = lib().bdsm_engine_apply_stream(self._h, parr, sarr, k, 1 if device else 0, _ptr(pos), _ptr(neg), stats,
                                           C.byref(done))
        out = [BatchResult(pos[i * nq:i * nq + self.nq].tolist(), neg[i * nq:i * nq + self.nq].tolist(),
                           _stats_dict(stats[i])) for i in range(done.value)]
        if r != 0:
            try:
                _raise(r, self._h)
            except Exception as e:  # the batches before the failing one were applied
                e.done = done.value
                e.results = out
                raise
        return out

    def match_stream(self, batches) -> List[BatchResult]:
        """Pipelined stream of host batches (bdsm_engine_apply_stream): the
        positive phase of batch i and the negative phase of batch i+1 share one
        matching launch; results equal one match_batch per batch.  On an error
        the exception carries .done (batches applied) and .results."""
        ups = [make_updates(b) for b in batches]
        return self._stream([u.ctypes.data for u in ups], [len(u) for u in ups], False)

    def match_stream_device(self, dev_ptrs, sizes) -> List[BatchResult]:
        """Same, with every batch already in device memory."""
        return self._stream(dev_ptrs, sizes, True)

    def set_deadline(self, query: int, seconds_from_now: float) -> None:
        r = lib().bdsm_engine_set_deadline(self._h, query, seconds_from_now)
        if r != 0:
            _raise(r, self._h)

    def set_query_active(self, query: int, active: bool) -> None:
        """Whether later batches match `query` (run_pipeline drops unsolved queries)."""
        r = lib().bdsm_engine_set_query_active(self._h, query, 1 if active else 0)
        if r != 0:
            _raise(r, self._h)

    def query_timed_out(self, query: int) -> bool:
        """MatchStats::timed_out of `query` in the last batch (its counts were dropped)."""
        r = lib().bdsm_engine_query_timed_out(self._h, query)
        if r < 0:
            _raise(-r, self._h)
        return r != 0

    def neighbors(self, v: int) -> List[int]:
        d = lib().bdsm_engine_neighbors(self._h, v, None, 0)
        out = np.zeros(max(d, 1), np.uint32)
        lib().bdsm_engine_neighbors(self._h, v, _ptr(out), d)
        return out[:d].tolist()

    def rows(self, query: int) -> np.ndarray:
        out = np.zeros(max(self.num_vertices, 1), np.uint32)
        r = lib().bdsm_engine_rows(self._h, query, _ptr(out))
        if r != 0:
            _raise(r, self._h)
        return out[: self.num_vertices]

    def order(self, query: int, edge: int) -> List[int]:
        out = np.zeros(32, np.uint32)
        n = lib().bdsm_engine_order(self._h, query, edge, _ptr(out))
        if n < 0:
            _raise(-n, self._h)
        return out[:n].tolist()

    def collect_matches(self, cap: int) -> None:
        """Materialise up to `cap` matches per (query, phase) for later batches (0: counts only)."""
        r = lib().bdsm_engine_collect_matches(self._h, cap)
        if r != 0:
            _raise(r, self._h)
        self._collect_cap = cap

    def matches(self, query: int, positive: bool) -> np.ndarray:
        """The last batch's matches of `query` (external ids, query vertex order, sorted)."""
        n = self.query_sizes[query]
        total = lib().bdsm_engine_matches(self._h, query, 1 if positive else 0, None, 0)
        if total < 0:
            _raise(int(-total), self._h)
        if total > getattr(self, "_collect_cap", 0):
            raise EngineError(3, f"{total} matches, only {getattr(self, '_collect_cap', 0)} collected "
                              "(raise the collect_matches cap)")
        out = np.zeros((total, n), np.uint32)
        got = lib().bdsm_engine_matches(self._h, query, 1 if positive else 0, _ptr(out), total)
        if got < 0:
            _raise(int(-got), self._h)
        return out

    def tail(self, query: int, edge: int) -> int:
        """First level of the independent tail of (query, edge)'s matching order."""
        t = lib().bdsm_engine_tail(self._h, query, edge)
        if t < 0:
            _raise(-t, self._h)
        return t

    def debug_trace(self) -> dict:
        """Per-phase matching-kernel trace of the last batch (-DBDSM_TRACE builds)."""
        out = np.zeros(32 + 64, np.uint64)
        lib().bdsm_engine_debug_trace(self._h, _ptr(out), out.size)
        names = ("busy_ns", "max_item_ns", "max_item", "static_items", "donated_items", "t_first", "t_last",
                 "mx_chunks", "mx_tail_chunks", "mx_big_leaf", "mx_donations", "mx_anchor_deg",
                 "mx_cy_donate", "mx_cy_filter", "mx_cy_leaf", "mx_cy_setup")
        r = {ph: dict(zip(names, out[16 * i: 16 * i + 16].tolist())) for i, ph in enumerate(("neg", "pos"))}
        for i, ph in enumerate(("neg", "pos")):
            r[ph]["chunks"] = out[32 + 16 * i: 48 + 16 * i].tolist()
            r[ph]["setups"] = out[64 + 16 * i: 80 + 16 * i].tolist()
        return r

    def column_sizes(self, query: int) -> List[int]:
        out = np.zeros(32, np.uint64)
        r = lib().bdsm_engine_column_sizes(self._h, query, _ptr(out))
        if r != 0:
            _raise(r, self._h)
        return out[: self.query_sizes[query]].tolist()

    def replan(self, query: int) -> None:
        r = lib().bdsm_engine_replan(self._h, query)
        if r != 0:
            _raise(r, self._h)

    @property
    def num_vertices(self) -> int:
        return int(lib().bdsm_engine_num_vertices(self._h))

    @property
    def num_edges(self) -> int:
        return int(lib().bdsm_engine_num_edges(self._h))

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().bdsm_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


class EngineGroup:
    """One engine per device in `devices` (a device may repeat), each holding a
    replica of the graph and counting its share of the work units
    (bdsm_group_*, SURVEY.md §8(e) in one process); counts are the sums over
    the engines and equal one Engine's."""

    def __init__(self, vertex_labels, src, dst, edge_labels=None, *, devices: Sequence[int] = (0,),
                 group_bits: int = 2, slack: float = 0.25, pool_reserve: float = 0.5, chunk: int = 32,
                 coalesce: bool = False):
        L = lib()
        self._vl = _u32(vertex_labels)
        s, d = _u32(src), _u32(dst)
        el = None if edge_labels is None else _u32(edge_labels)
        desc = _GraphDesc(len(self._vl), self._vl.ctypes.data, len(s), s.ctypes.data, d.ctypes.data,
                          None if el is None else el.ctypes.data)
        opts = _Options(group_bits, 1 if coalesce else 0, 0, 0, 1, slack, pool_reserve, chunk, 0, 0)
        devs = np.ascontiguousarray(np.asarray(list(devices), dtype=np.int32))
        h = C.c_void_p()
        st = L.bdsm_group_create(C.byref(desc), C.byref(opts), devs.ctypes.data, len(devs), C.byref(h))
        if st != 0:
            _raise(st)
        self._h = h
        self.nq = 0
        self.query_sizes: List[int] = []

    def _e0(self):
        return lib().bdsm_group_engine(self._h, 0)

    @property
    def size(self) -> int:
        return int(lib().bdsm_group_size(self._h))

    def add_query(self, labels: Sequence[int], edges: Iterable[Tuple]) -> int:
        ql = _u32(labels)
        edges = list(edges)
        qa = _u32([e[0] for e in edges])
        qb = _u32([e[1] for e in edges])
        qlab = _u32([NO_LABEL if (len(e) < 3 or e[2] is None or e[2] < 0) else e[2] for e in edges])
        desc = _QueryDesc(len(ql), ql.ctypes.data, len(qa), qa.ctypes.data if len(qa) else None,
                          qb.ctypes.data if len(qb) else None, qlab.ctypes.data if len(qlab) else None)
        r = lib().bdsm_group_add_query(self._h, C.byref(desc))
        if r < 0:
            _raise(-r)
        self.nq += 1
        self.query_sizes.append(len(ql))
        return r

    def match_batch(self, updates) -> BatchResult:
        ups = make_updates(updates)
        pos = np.zeros(max(self.nq, 1), np.uint64)
        neg = np.zeros(max(self.nq, 1), np.uint64)
        st = _Stats()
        r = lib().bdsm_group_apply_batch(self._h, _ptr(ups) if len(ups) else None, len(ups), _ptr(pos), _ptr(neg),
                                         C.byref(st))
        if r != 0:
            _raise(r, self._e0())
        return BatchResult(pos[: self.nq].tolist(), neg[: self.nq].tolist(), _stats_dict(st))

    def match_stream(self, batches) -> List[BatchResult]:
        ups = [make_updates(b) for b in batches]
        k, nq = len(ups), max(self.nq, 1)
        parr = (C.c_void_p * max(k, 1))(*[C.c_void_p(u.ctypes.data) for u in ups])
        sarr = (C.c_size_t * max(k, 1))(*[len(u) for u in ups])
        pos = np.zeros(max(k * nq, 1), np.uint64)
        neg = np.zeros(max(k * nq, 1), np.uint64)
        stats = (_Stats * max(k, 1))()
        done = C.c_size_t(0)
        r = lib().bdsm_group_apply_stream(self._h, parr, sarr, k, _ptr(pos), _ptr(neg), stats, C.byref(done))
        out = [BatchResult(pos[i * nq:i * nq + self.nq].tolist(), neg[i * nq:i * nq + self.nq].tolist(),
                           _stats_dict(stats[i])) for i in range(done.value)]
        if r != 0:
            try:
                _raise(r, self._e0())
            except Exception as e:
                e.done = done.value
                e.results = out
                raise
        return out

    def set_query_active(self, query: int, active: bool) -> None:
        r = lib().bdsm_group_set_query_active(self._h, query, 1 if active else 0)
        if r != 0:
            _raise(r)

    def collect_matches(self, cap: int) -> None:
        r = lib().bdsm_group_collect_matches(self._h, cap)
        if r != 0:
            _raise(r)
        self._collect_cap = cap

    def matches(self, query: int, positive: bool) -> np.ndarray:
        """The last batch's matches of `query` over every engine, merged and sorted."""
        n = self.query_sizes[query]
        total = lib().bdsm_group_matches(self._h, query, 1 if positive else 0, None, 0)
        if total < 0:
            _raise(int(-total))
        if total > getattr(self, "_collect_cap", 0):  # as Engine.matches: the cap bounds the total
            raise EngineError(3, f"{total} matches, only {getattr(self, '_collect_cap', 0)} collected "
                              "(raise the collect_matches cap)")
        out = np.zeros((total, n), np.uint32)
        got = lib().bdsm_group_matches(self._h, query, 1 if positive else 0, _ptr(out), total)
        if got < 0:
            _raise(int(-got))
        return out

    def neighbors(self, v: int, replica: int = 0) -> List[int]:
        e = lib().bdsm_group_engine(self._h, replica)
        d = lib().bdsm_engine_neighbors(e, v, None, 0)
        out = np.zeros(max(d, 1), np.uint32)
        lib().bdsm_engine_neighbors(e, v, _ptr(out), d)
        return out[:d].tolist()

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().bdsm_group_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def plan_edge_orbits(labels: Sequence[int], edges) -> Tuple[List[int], int]:
    """Exact-coalescing plan of a query (host only): per directed edge
    d = 2*edge + flip the multiplicity its search stands for (orbit size for an
    orbit's representative, 0 for the others), and the automorphism count
    (0: more than 20,000, no coalescing)."""
    L = lib()
    lab = np.ascontiguousarray(np.asarray(labels, dtype=np.uint32))
    ea = np.ascontiguousarray(np.asarray([e[0] for e in edges], dtype=np.uint32))
    eb = np.ascontiguousarray(np.asarray([e[1] for e in edges], dtype=np.uint32))
    desc = _QueryDesc(len(lab), _ptr(lab), len(ea), _ptr(ea), _ptr(eb), None)
    mult = np.zeros(max(2 * len(ea), 1), np.uint32)
    r = L.bdsm_plan_edge_orbits(C.byref(desc), _ptr(mult))
    if r < 0:
        _raise(int(-r))
    return mult[:2 * len(ea)].tolist(), int(r)


def shard_owners(costs: Sequence[int], world: int) -> List[int]:
    """Owner rank of each work unit (canonical order) under the cost-balanced
    split used by the engine: floor(world * prefix / total)."""
    c = np.ascontiguousarray(np.asarray(costs, dtype=np.uint64))
    out = np.zeros(max(len(c), 1), np.uint32)
    lib().bdsm_shard_owners(_ptr(c), len(c), world, _ptr(out))
    return out[: len(c)].tolist()


def version() -> str:
    return lib().bdsm_version().decode()

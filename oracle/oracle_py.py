"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the CPU restatement
(oracle/liboracle.so, see oracle.hpp) and for the reference shim
(oracle/_ref/libbdsm_refshim.so, see ref_shim.cpp).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg import
this module, and only as the checker.  The product package
(paper_2401_17018_b200) never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
NONE = 0xFFFFFFFF

_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")

_lib = None
_ref = None


def build(ref: bool = False) -> None:
    """Compile the restatement (and, when /root/reference exists, the reference)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    if ref and os.path.isdir("/root/reference/proj"):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        L.orc_create.restype = C.c_void_p
        L.orc_create.argtypes = [C.c_uint32, _u32p, C.c_uint64, _u32p, _u32p, C.c_void_p,
                                 C.c_uint32, C.c_char_p, C.c_size_t]
        L.orc_add_query.restype = C.c_int
        L.orc_add_query.argtypes = [C.c_void_p, C.c_uint32, _u32p, C.c_uint32, _u32p, _u32p,
                                    C.c_void_p, C.c_char_p, C.c_size_t]
        L.orc_apply_batch.restype = C.c_int
        L.orc_apply_batch.argtypes = [C.c_void_p, C.c_uint64, _u32p, _u32p, _u8p, C.c_void_p,
                                      C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p,
                                      C.c_void_p, C.c_char_p, C.c_size_t]
        L.orc_last_errors.restype = C.c_size_t
        L.orc_last_errors.argtypes = [C.c_void_p, _u64p, _u32p, C.c_size_t]
        L.orc_order.restype = C.c_int
        L.orc_order.argtypes = [C.c_void_p, C.c_int, C.c_uint32, _u32p, C.c_size_t]
        L.orc_row.restype = C.c_uint32
        L.orc_row.argtypes = [C.c_void_p, C.c_int, C.c_uint32]
        L.orc_degree.restype = C.c_uint64
        L.orc_degree.argtypes = [C.c_void_p, C.c_uint32]
        L.orc_destroy.restype = None
        L.orc_destroy.argtypes = [C.c_void_p]
        _lib = L
    return _lib


def _arr(x, dt=np.uint32):
    return np.ascontiguousarray(np.asarray(x, dtype=dt))


def _opt_ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class OracleError(Exception):
    def __init__(self, status: int, msg: str, failures=None):
        super().__init__(msg)
        self.status = status
        self.failures = failures or []


class Oracle:
    """Count-only CPU restatement of bdsm::match_batch (coalesce off)."""

    def __init__(self, vlabels, eu, ev, elab=None, group_bits: int = 2):
        L = lib()
        self._vl = _arr(vlabels)
        eu, ev = _arr(eu), _arr(ev)
        self._elab = None if elab is None else _arr(elab)
        err = C.create_string_buffer(512)
        self.h = L.orc_create(len(self._vl), self._vl, len(eu), eu, ev, _opt_ptr(self._elab),
                              group_bits, err, 512)
        if not self.h:
            raise OracleError(2, err.value.decode())
        self.nq = 0

    def add_query(self, qlabels, qedges) -> int:
        """qedges: iterable of (a, b, label or None/-1)."""
        ql = _arr(qlabels)
        qa = _arr([e[0] for e in qedges])
        qb = _arr([e[1] for e in qedges])
        qlab = _arr([NONE if (len(e) < 3 or e[2] is None or e[2] < 0) else e[2] for e in qedges])
        err = C.create_string_buffer(512)
        r = lib().orc_add_query(self.h, len(ql), ql, len(qa), qa, qb, _opt_ptr(qlab), err, 512)
        if r < 0:
            raise OracleError(-r, err.value.decode())
        self.nq += 1
        return r

    def apply_batch(self, updates, nthreads: int = 1, rank: int = 0, world: int = 1,
                    match: bool = True):
        """updates: iterable of (op, u, v[, label]) with op 0 insert / 1 delete.
        Returns (pos[nq], neg[nq], stats[7])."""
        ups = list(updates)
        uop = _arr([u[0] for u in ups], np.uint8)
        uu = _arr([u[1] for u in ups])
        uv = _arr([u[2] for u in ups])
        ul = _arr([NONE if (len(u) < 4 or u[3] is None or u[3] < 0) else u[3] for u in ups])
        pos = np.zeros(max(1, self.nq), np.uint64)
        neg = np.zeros(max(1, self.nq), np.uint64)
        st = np.zeros(7, np.uint64)
        err = C.create_string_buffer(512)
        r = lib().orc_apply_batch(self.h, len(ups), uu, uv, uop, _opt_ptr(ul), nthreads, rank, world,
                                  _opt_ptr(pos) if match else None, _opt_ptr(neg) if match else None,
                                  _opt_ptr(st), err, 512)
        if r != 0:
            fails = []
            if r == 1:
                idx = np.zeros(len(ups), np.uint64)
                code = np.zeros(len(ups), np.uint32)
                k = lib().orc_last_errors(self.h, idx, code, len(ups))
                fails = list(zip(idx[:k].tolist(), code[:k].tolist()))
            raise OracleError(r, err.value.decode(), fails)
        return pos[: self.nq].tolist(), neg[: self.nq].tolist(), st.tolist()

    def order(self, q: int, e: int):
        out = np.zeros(32, np.uint32)
        n = lib().orc_order(self.h, q, e, out, 32)
        return out[:n].tolist()

    def row(self, q: int, v: int) -> int:
        return int(lib().orc_row(self.h, q, v))

    def degree(self, v: int) -> int:
        return int(lib().orc_degree(self.h, v))

    def close(self):
        if self.h:
            lib().orc_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# --------------------------------------------------------------------------
# Reference shim (only where oracle/_ref was built; absent on a box without it)

def ref_available() -> bool:
    return os.path.exists(os.path.join(HERE, "_ref", "libbdsm_refshim.so"))


def ref():
    global _ref
    if _ref is None:
        L = C.CDLL(os.path.join(HERE, "_ref", "libbdsm_refshim.so"))
        L.ref_run_stream.restype = C.c_int
        L.ref_run_stream.argtypes = [
            C.c_uint32, _u32p, C.c_uint64, _u32p, _u32p, C.c_void_p,
            C.c_uint32, _u32p, C.c_uint32, _u32p, _u32p, C.c_void_p,
            C.c_uint32, _u64p, _u32p, _u32p, _u8p, C.c_void_p,
            C.c_uint32, C.c_int, C.c_uint32, _u64p, _u64p, _u64p, _f64p, _u64p,
            C.c_void_p, C.c_void_p, C.c_char_p, C.c_size_t]
        L.ref_oracle_diff.restype = C.c_int
        L.ref_oracle_diff.argtypes = [
            C.c_uint32, _u32p, C.c_uint64, _u32p, _u32p, C.c_void_p,
            C.c_uint32, _u32p, C.c_uint32, _u32p, _u32p, C.c_void_p,
            C.c_uint64, _u32p, _u32p, _u8p, C.c_void_p, _u64p, _u64p, C.c_char_p, C.c_size_t]
        L.ref_plan_orders.restype = C.c_int
        L.ref_plan_orders.argtypes = [
            C.c_uint32, _u32p, C.c_uint64, _u32p, _u32p, C.c_void_p,
            C.c_uint32, _u32p, C.c_uint32, _u32p, _u32p, C.c_void_p, C.c_uint32, _u32p, _u64p,
            C.c_char_p, C.c_size_t]
        _ref = L
    return _ref


def ref_plan_orders(vlabels, eu, ev, elab, qlabels, qedges, group_bits: int = 2):
    """The UNMODIFIED reference's plan with coalescing off: (orders per query
    edge, candidate column sizes it was built from)."""
    vl, eu, ev = _arr(vlabels), _arr(eu), _arr(ev)
    el = None if elab is None else _arr(elab)
    ql = _arr(qlabels)
    qa = _arr([e[0] for e in qedges])
    qb = _arr([e[1] for e in qedges])
    qlab = _arr([NONE if (len(e) < 3 or e[2] is None or e[2] < 0) else e[2] for e in qedges])
    orders = np.zeros(32 * max(len(qa), 1), np.uint32)
    cols = np.zeros(max(len(ql), 1), np.uint64)
    err = C.create_string_buffer(512)
    r = ref().ref_plan_orders(len(vl), vl, len(eu), eu, ev, _opt_ptr(el), len(ql), ql, len(qa), qa, qb,
                              _opt_ptr(qlab), group_bits, orders, cols, err, 512)
    if r != 0:
        raise OracleError(r, err.value.decode())
    n = len(ql)
    return [orders[32 * e: 32 * e + n].tolist() for e in range(len(qa))], cols[:n].tolist()


def ref_run_stream(vlabels, eu, ev, elab, qlabels, qedges, batches: Sequence, workers: int = 1,
                   plan_mode: int = 0, group_bits: int = 2):
    """Runs the UNMODIFIED reference match_batch over a stream.  Returns a list
    of (pos, neg, visits) per batch and [visits, iops, tasks, emitted]."""
    vl, eu, ev = _arr(vlabels), _arr(eu), _arr(ev)
    el = None if elab is None else _arr(elab)
    ql = _arr(qlabels)
    qa = _arr([e[0] for e in qedges])
    qb = _arr([e[1] for e in qedges])
    qlab = _arr([NONE if (len(e) < 3 or e[2] is None or e[2] < 0) else e[2] for e in qedges])
    flat = [u for b in batches for u in b]
    offs = _arr(np.cumsum([0] + [len(b) for b in batches]), np.uint64)
    uop = _arr([u[0] for u in flat], np.uint8)
    uu = _arr([u[1] for u in flat])
    uv = _arr([u[2] for u in flat])
    ul = _arr([NONE if (len(u) < 4 or u[3] is None or u[3] < 0) else u[3] for u in flat])
    nb = len(batches)
    pos, neg, vis = (np.zeros(max(nb, 1), np.uint64) for _ in range(3))
    ms = np.zeros(max(nb, 1), np.float64)
    st = np.zeros(4, np.uint64)
    err = C.create_string_buffer(512)
    r = ref().ref_run_stream(len(vl), vl, len(eu), eu, ev, _opt_ptr(el), len(ql), ql, len(qa), qa, qb,
                             _opt_ptr(qlab), nb, offs, uu, uv, uop, _opt_ptr(ul), workers, plan_mode,
                             group_bits, pos, neg, vis, ms, st, None, None, err, 512)
    if r != 0:
        raise OracleError(r, err.value.decode())
    return [(int(pos[i]), int(neg[i]), int(vis[i])) for i in range(nb)], st.tolist()

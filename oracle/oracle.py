"""ORACLE — TEST INFRASTRUCTURE ONLY (never the product path).

ctypes front end of ``oracle/_ref/libqbref.so``: the reference's own C++ kernels,
containers and RNG (compiled in place from /root/reference/proj/src by
oracle/Makefile) plus the restated algorithm layer (oracle/qr_restated.cpp,
oracle/qb_restated.cpp) that the reference snapshot is missing.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline
leg may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libqbref.so")
REFERENCE_SRC = "/root/reference/proj"

TERMINATION = {0: "rank_reached", 1: "tolerance_met", 2: "sketch_exhausted", 3: "rank_collapse"}
STATUS = {0: "ok", 1: "DimensionError", 2: "SingularityError", 3: "ToleranceFloorError",
          4: "FormatError", 5: "ResourceError", 6: "Error", 7: "other"}
ALG = {"ei": 0, "fp": 1, "fp_fixed_rank": 2, "single_pass": 3, "qb": 4, "qb_b": 5, "arf": 6}


class QboParams(C.Structure):
    _fields_ = [("alg", C.c_int32), ("mode", C.c_int32),
                ("b", C.c_int64), ("power", C.c_int64), ("k", C.c_int64), ("s", C.c_int64),
                ("max_rank", C.c_int64), ("l_budget", C.c_int64), ("max_restarts", C.c_int64),
                ("eps_abs", C.c_double), ("seed", C.c_uint64), ("stream", C.c_uint64),
                ("reorth", C.c_int32), ("pad_", C.c_int32)]


class QboResult(C.Structure):
    _fields_ = [("rank", C.c_int64), ("E", C.c_double), ("norm_a_sq", C.c_double),
                ("passes", C.c_int64), ("terminated_by", C.c_int32), ("status", C.c_int32),
                ("diag_index", C.c_int64), ("floor", C.c_double), ("m", C.c_int64),
                ("n", C.c_int64), ("n_trace", C.c_int64), ("msg", C.c_char * 256),
                ("seconds", C.c_double)]


def build(force: bool = False) -> str:
    """Compile oracle/_ref/libqbref.so when the reference sources are present."""
    if os.path.isdir(REFERENCE_SRC) and (force or not os.path.exists(LIB_PATH)):
        subprocess.check_call(["make", "-s", "-j8", "-C", HERE])
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        P, I64, U64, D = C.c_void_p, C.c_int64, C.c_uint64, C.c_double
        L.qbo_lane_name.restype = C.c_char_p
        L.qbo_rng_u64.argtypes = [U64, U64, I64, P]
        L.qbo_rng_double.argtypes = [U64, U64, I64, P]
        L.qbo_gaussian.argtypes = [U64, U64, I64, I64, I64, P]
        L.qbo_substream_id.argtypes = [U64, U64, U64, P]
        L.qbo_orth_qr.argtypes = [I64, I64, P, P, P]
        L.qbo_rank_deficiency.argtypes = [I64, P, D, P, P]
        L.qbo_tri_solve_t.argtypes = [I64, I64, P, P, P, D, P]
        L.qbo_orth_loss.argtypes = [I64, I64, P]
        L.qbo_orth_loss.restype = D
        L.qbo_validate_epsilon.argtypes = [D, D, D, P]
        L.qbo_dense_multiply.argtypes = [I64, I64, P, I64, P, C.c_int, P]
        L.qbo_csr_multiply.argtypes = [I64, I64, I64, P, P, P, I64, P, C.c_int, P]
        L.qbo_csr_frob_sq.argtypes = [I64, I64, I64, P, P, P]
        L.qbo_csr_frob_sq.restype = D
        L.qbo_csr_validate.argtypes = [I64, I64, I64, P, P, P, I64]
        L.qbo_csr_from_triplets.argtypes = [I64, I64, I64, P, P, P, P, P, P]
        L.qbo_run_dense.argtypes = [I64, I64, P, P, P]
        L.qbo_run_dense.restype = P
        L.qbo_run_csr.argtypes = [I64, I64, I64, P, P, P, P, P]
        L.qbo_run_csr.restype = P
        L.qbo_copy_q.argtypes = [P, P]
        L.qbo_copy_b.argtypes = [P, P]
        L.qbo_copy_trace.argtypes = [P, P]
        L.qbo_free.argtypes = [P]
        L.qbo_explicit_error_dense.argtypes = [I64, I64, P, I64, P, P]
        L.qbo_explicit_error_dense.restype = D
        L.qbo_explicit_error_csr.argtypes = [I64, I64, I64, P, P, P, I64, P, P]
        L.qbo_explicit_error_csr.restype = D
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _f64(a):
    return np.asfortranarray(a, dtype=np.float64)


def lane_name() -> str:
    return lib().qbo_lane_name().decode()


# ---- RNG (rng.cpp:28-79) ----------------------------------------------------
def rng_u64(seed: int, count: int, stream: int = 0) -> np.ndarray:
    out = np.empty(count, dtype=np.uint64)
    lib().qbo_rng_u64(seed, stream, count, _p(out))
    return out


def rng_double(seed: int, count: int, stream: int = 0) -> np.ndarray:
    out = np.empty(count, dtype=np.float64)
    lib().qbo_rng_double(seed, stream, count, _p(out))
    return out


def gaussian(rows: int, cols: int, seed: int, stream: int = 0, skip: int = 0) -> np.ndarray:
    out = np.empty((rows, cols), dtype=np.float64, order="F")
    st = lib().qbo_gaussian(seed, stream, skip, rows, cols, _p(out))
    if st:
        raise ValueError(STATUS[st])
    return out


def substream_id(seed: int, stream: int, sub: int) -> int:
    out = np.zeros(1, dtype=np.uint64)
    lib().qbo_substream_id(seed, stream, sub, _p(out))
    return int(out[0])


# ---- primitives (qr.hpp:10-29) ---------------------------------------------
def orth_qr(a):
    a = _f64(a)
    m, n = a.shape
    q = np.empty((m, n), order="F")
    r = np.empty((n, n), order="F")
    st = lib().qbo_orth_qr(m, n, _p(a), _p(q), _p(r))
    if st:
        raise ValueError(STATUS[st])
    return q, r


def rank_deficiency_report(r, threshold=1e-12):
    r = _f64(r)
    n = r.shape[0]
    out = np.zeros(max(n, 1), dtype=np.int64)
    cnt = np.zeros(1, dtype=np.int64)
    lib().qbo_rank_deficiency(n, _p(r), threshold, _p(out), _p(cnt))
    return [int(x) for x in out[: int(cnt[0])]]


def tri_solve_transposed(r, c, threshold=1e-12):
    r, c = _f64(r), _f64(c)
    x = np.empty_like(c, order="F")
    di = np.zeros(1, dtype=np.int64)
    st = lib().qbo_tri_solve_t(r.shape[0], c.shape[1], _p(r), _p(c), _p(x), threshold, _p(di))
    return st, int(di[0]), x


def orthogonality_loss(q) -> float:
    q = _f64(q)
    return lib().qbo_orth_loss(q.shape[0], q.shape[1], _p(q))


def validate_epsilon(eps, frob_a, delta=0.01):
    fl = np.zeros(1)
    ok = lib().qbo_validate_epsilon(eps, frob_a, delta, _p(fl))
    return bool(ok), float(fl[0])


def dense_multiply(a, x, trans=False):
    a, x = _f64(a), _f64(x)
    m, n = a.shape
    y = np.empty((n if trans else m, x.shape[1]), order="F")
    st = lib().qbo_dense_multiply(m, n, _p(a), x.shape[1], _p(x), int(trans), _p(y))
    if st:
        raise ValueError(STATUS[st])
    return y


def _csr_arrays(csr):
    m, n, rp, ci, v = csr
    return (int(m), int(n), np.ascontiguousarray(rp, dtype=np.int64),
            np.ascontiguousarray(ci, dtype=np.int32), np.ascontiguousarray(v, dtype=np.float64))


def csr_multiply(csr, x, trans=False):
    m, n, rp, ci, v = _csr_arrays(csr)
    x = _f64(x)
    y = np.empty((n if trans else m, x.shape[1]), order="F")
    st = lib().qbo_csr_multiply(m, n, len(v), _p(rp), _p(ci), _p(v), x.shape[1], _p(x),
                                int(trans), _p(y))
    if st:
        raise ValueError(STATUS[st])
    return y


def csr_frob_sq(csr) -> float:
    m, n, rp, ci, v = _csr_arrays(csr)
    return lib().qbo_csr_frob_sq(m, n, len(v), _p(rp), _p(ci), _p(v))


def csr_validate(m, n, rp, ci, v) -> str:
    rp = np.ascontiguousarray(rp, dtype=np.int64)
    ci = np.ascontiguousarray(ci, dtype=np.int32)
    v = np.ascontiguousarray(v, dtype=np.float64)
    return STATUS[lib().qbo_csr_validate(m, n, len(v), _p(rp), _p(ci), _p(v), len(rp))]


def csr_from_triplets(m, n, rows, cols, vals):
    """SparseCsrMatrix::from_triplets (sparse_csr.cpp:42-64) -> (status, rp, ci, v)."""
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    cols = np.ascontiguousarray(cols, dtype=np.int64)
    vals = np.ascontiguousarray(vals, dtype=np.float64)
    rp = np.zeros(m + 1, dtype=np.int64)
    ci = np.zeros(max(len(vals), 1), dtype=np.int32)
    v = np.zeros(max(len(vals), 1), dtype=np.float64)
    st = lib().qbo_csr_from_triplets(m, n, len(vals), _p(rows), _p(cols), _p(vals), _p(rp), _p(ci), _p(v))
    return STATUS[st], rp, ci[:len(vals)], v[:len(vals)]


# ---- algorithms ----------------------------------------------------------------
@dataclass
class OracleQB:
    Q: np.ndarray
    B: np.ndarray
    rank: int
    E: float
    norm_a_sq: float
    passes: int
    terminated_by: str
    e_trace: np.ndarray
    seconds: float = 0.0  # steady_clock around the rand_qb_* call inside the oracle


class OracleError(Exception):
    def __init__(self, status, msg, diag_index=0, floor=0.0):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = STATUS.get(status, str(status))
        self.diag_index = diag_index
        self.floor = floor


def run(alg: str, a=None, csr=None, *, b=10, power=0, eps_abs=0.0, fixed_rank=None,
        max_rank=0, l_budget=0, max_restarts=8, seed=0, stream=0, reorth=True) -> OracleQB:
    p = QboParams()
    p.alg = ALG[alg]
    p.mode = 0 if fixed_rank is not None else 1
    k, s = fixed_rank if fixed_rank is not None else (0, 0)
    p.b, p.power, p.k, p.s = b, power, k, s
    p.max_rank, p.l_budget, p.max_restarts = max_rank, l_budget, max_restarts
    p.eps_abs, p.seed, p.stream, p.reorth = eps_abs, seed, stream, int(reorth)
    res = QboResult()
    L = lib()
    if csr is not None:
        m, n, rp, ci, v = _csr_arrays(csr)
        h = L.qbo_run_csr(m, n, len(v), _p(rp), _p(ci), _p(v), C.byref(p), C.byref(res))
    else:
        a = _f64(a)
        m, n = a.shape
        h = L.qbo_run_dense(m, n, _p(a), C.byref(p), C.byref(res))
    if res.status:
        raise OracleError(res.status, res.msg.decode(), res.diag_index, res.floor)
    r = int(res.rank)
    Q = np.empty((m, r), order="F")
    B = np.empty((r, n), order="F")
    tr = np.empty(int(res.n_trace))
    if r:
        L.qbo_copy_q(h, _p(Q))
        L.qbo_copy_b(h, _p(B))
    if res.n_trace:
        L.qbo_copy_trace(h, _p(tr))
    L.qbo_free(h)
    return OracleQB(Q, B, r, res.E, res.norm_a_sq, int(res.passes),
                    TERMINATION[res.terminated_by], tr, float(res.seconds))


def explicit_error(q, b, a=None, csr=None) -> float:
    q, b = _f64(q), _f64(b)
    k = q.shape[1]
    if csr is not None:
        m, n, rp, ci, v = _csr_arrays(csr)
        return lib().qbo_explicit_error_csr(m, n, len(v), _p(rp), _p(ci), _p(v), k, _p(q), _p(b))
    a = _f64(a)
    return lib().qbo_explicit_error_dense(a.shape[0], a.shape[1], _p(a), k, _p(q), _p(b))

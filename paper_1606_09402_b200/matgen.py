"""Synthetic inputs for the BASELINE configs (harness side, not the product path).

The reference's generator (src/matgen.cpp) is missing from the
snapshot; the recipes here are the builder's, recorded in DESIGN.md §Inputs and
SURVEY.md §8(d). Gaussians come from this repo's own host RNG (libqbfac_matgen.so,
stream-compatible with the reference RngStream) or, for large inputs on a GPU box,
from the device generator of libqbfac_gpu.so; QR factors are computed with numpy
(LAPACK) or torch (cuSOLVER) with the diag(R) >= 0 sign convention of qr.hpp:15-18.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_mg = None


def mglib():
    global _mg
    if _mg is None:
        path = os.path.join(HERE, "libqbfac_matgen.so")
        if not os.path.exists(path):
            raise ImportError(f"{path} missing; run __graft_entry__.build()")
        L = C.CDLL(path)
        P, I64, U64, D = C.c_void_p, C.c_int64, C.c_uint64, C.c_double
        L.qbm_gaussian.argtypes = [U64, U64, I64, I64, P]
        L.qbm_u64.argtypes = [U64, U64, I64, P]
        L.qbm_gaussian_add.argtypes = [U64, U64, I64, I64, D, P]
        L.qbm_csr_uniform.argtypes = [U64, I64, I64, I64, P, P, P]
        L.qbm_csr_zipf.argtypes = [U64, I64, I64, D, D, P, P, P]
        L.qbm_csr_zipf.restype = I64
        _mg = L
    return _mg


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def host_gaussian(rows: int, cols: int, seed: int, stream: int = 0, skip: int = 0) -> np.ndarray:
    out = np.empty(rows * cols)
    mglib().qbm_gaussian(seed, stream, skip, rows * cols, _p(out))
    return out.reshape((rows, cols), order="F")


def host_u64(seed: int, count: int, stream: int = 0) -> np.ndarray:
    out = np.empty(count, dtype=np.uint64)
    mglib().qbm_u64(seed, stream, count, _p(out))
    return out


# ---- spectra --------------------------------------------------------
def spectrum(kind: str, n: int, **kw) -> np.ndarray:
    j = np.arange(1, n + 1, dtype=np.float64)
    if kind == "inv_square":
        return 1.0 / j**2
    if kind == "inv":
        return 1.0 / j
    if kind == "exp_decay":
        return np.exp(-j / kw.get("tau", 7.0))
    if kind == "pow10":  # cfg1: 10^(-j/200)
        return 10.0 ** (-j / kw.get("scale", 200.0))
    if kind == "s_shape":
        e = np.clip(j - kw.get("center", 30), -700, 700)
        return kw.get("floor", 1e-4) + 1.0 / (1.0 + np.exp(e))
    raise ValueError(kind)


def optimal_rank(sigma: np.ndarray, eps_rel: float) -> int:
    """Smallest k with (sum_{j>k} s_j^2)^(1/2) < eps_rel * ||s||."""
    s2 = np.asarray(sigma, dtype=np.float64) ** 2
    total = s2.sum()
    tail = total - np.cumsum(s2)  # tail[k-1] = sum_{j>k}
    thr = (eps_rel**2) * total
    tails = np.concatenate([[total], tail])
    for k in range(len(tails)):
        if tails[k] < thr:
            return k
    return len(sigma)


def qr_pos(a: np.ndarray) -> np.ndarray:
    """Q of the economic QR with diag(R) >= 0 (qr.hpp:15-18)."""
    q, r = np.linalg.qr(a)
    sg = np.sign(np.diag(r))
    sg[sg == 0] = 1.0
    return np.asfortranarray(q * sg)


# ---- dense configs ------------------------------------------------------------------------
def synthesize(m: int, n: int, sigma: np.ndarray, seed: int) -> np.ndarray:
    """A = U diag(sigma) V^T with U, V the Q factors of gaussian(m, r) then gaussian(n, r)
    drawn from one RngStream(seed) (r = len(sigma))."""
    r = len(sigma)
    gu = host_gaussian(m, r, seed, 0, 0)
    gv = host_gaussian(n, r, seed, 0, m * r)
    u = qr_pos(gu)
    v = qr_pos(gv)
    return np.asfortranarray((u * sigma) @ v.T)


def synthesize_torch(m: int, n: int, sigma: np.ndarray, seed: int, noise: float = 0.0, device="cuda"):
    """Same recipe on the GPU (torch + cuSOLVER QR) with device-generated gaussians; returns
    a column-major (Fortran-ordered) torch tensor view A (m x n) as A_t^T storage."""
    import torch
    from .qbfac import default_context, lib

    ctx = default_context()
    r = len(sigma)

    def dev_gauss(rows, cols, stream, skip):
        t = torch.empty((cols, rows), dtype=torch.float64, device=device)  # column-major rows x cols
        # the library writes on its own stream: torch's pending work on this (possibly just
        # recycled) block must finish first
        torch.cuda.synchronize()
        ctx.check(lib().qbfac_gpu_gaussian_device(ctx.handle, seed, stream, skip, rows, cols,
                                                  C.c_void_p(t.data_ptr()), rows))
        ctx.synchronize()
        return t.t()  # rows x cols view

    def qpos(g):
        q, rr = torch.linalg.qr(g)
        sg = torch.sign(torch.diagonal(rr))
        sg[sg == 0] = 1.0
        return q * sg

    u = qpos(dev_gauss(m, r, 0, 0))
    v = qpos(dev_gauss(n, r, 0, m * r))
    sig = torch.as_tensor(sigma, dtype=torch.float64, device=device)
    at = (v * sig) @ u.t()  # n x m row-major == A column-major
    if noise:
        nz = dev_gauss(m, n, 1, 0)  # separate substream for the noise
        at += noise * nz.t()
    torch.cuda.synchronize()
    return at  # at.t() is A; at is contiguous (A column-major)


@dataclass
class Config:
    name: str
    alg: str
    m: int
    n: int
    b: int
    power: int
    eps_rel: float
    max_rank: int
    l_budget: int = 0
    sparse: bool = False
    omega_seed: int = 42


CONFIGS = {
    1: Config("cfg1_ei_dense_2000", "ei", 2000, 2000, 20, 0, 1e-2, 1000),
    2: Config("cfg2_fp_dense_8000", "fp", 8000, 8000, 50, 1, 5e-2, 2000, l_budget=2000),
    3: Config("cfg3_ei_csr_1e5x5e4", "ei", 100000, 50000, 50, 1, 0.5, 1000, sparse=True),
    4: Config("cfg4_fp_single_pass_40000x20000", "single_pass", 40000, 20000, 100, 0, 0.0, 400),
    5: Config("cfg5_ei_csr_zipf_2e6x5e5", "ei", 2000000, 500000, 100, 2, 0.6, 2000, sparse=True),
}


def cfg1_matrix(n: int = 2000, seed: int = 1) -> np.ndarray:
    return synthesize(n, n, spectrum("pow10", n), seed)


def cfg2_matrix(n: int = 8000, seed: int = 2) -> np.ndarray:
    return synthesize(n, n, spectrum("inv", n), seed)


def cfg4_matrix(m: int = 40000, n: int = 20000, r: int = 400, seed: int = 4, noise: float = 1e-6) -> np.ndarray:
    sig = np.exp(-np.arange(1, r + 1) / 60.0)
    a = synthesize(m, n, sig, seed)
    if noise:
        a += noise * host_gaussian(m, n, seed, 1, 0)
    return a


def csr_uniform(m: int, n: int, per_row: int, seed: int = 3):
    rp = np.empty(m + 1, dtype=np.int64)
    ci = np.empty(m * per_row, dtype=np.int32)
    v = np.empty(m * per_row, dtype=np.float64)
    st = mglib().qbm_csr_uniform(seed, m, n, per_row, _p(rp), _p(ci), _p(v))
    if st:
        raise ValueError("per_row > n")
    return m, n, rp, ci, v


def csr_zipf(m: int, n: int, alpha: float = 1.1, target_nnz: float = 2e8, seed: int = 5, c: float = 0.0):
    if not c:
        # c so that sum_r min(n, c r^-alpha) ~ target (before de-duplication)
        r = np.arange(1, m + 1, dtype=np.float64)
        lo, hi = 1.0, 1e12
        for _ in range(100):
            mid = math.sqrt(lo * hi)
            tot = np.minimum(n, np.maximum(1.0, np.round(mid * r**-alpha))).sum()
            lo, hi = (mid, hi) if tot < target_nnz else (lo, mid)
        c = math.sqrt(lo * hi)
    L = mglib()
    nnz = L.qbm_csr_zipf(seed, m, n, alpha, c, None, None, None)
    rp = np.empty(m + 1, dtype=np.int64)
    ci = np.empty(nnz, dtype=np.int32)
    v = np.empty(nnz, dtype=np.float64)
    L.qbm_csr_zipf(seed, m, n, alpha, c, _p(rp), _p(ci), _p(v))
    return m, n, rp, ci, v


def csr_to_dense(csr) -> np.ndarray:
    m, n, rp, ci, v = csr
    a = np.zeros((m, n), order="F")
    rows = np.repeat(np.arange(m), np.diff(rp))
    a[rows, ci] = v
    return a

"""Bit-reproducible dense inputs for BASELINE configs 2 and 4 (harness side, not the
product path).

The recipe: A = U diag(sigma) V^T, U and V the Q factors (diag(R) >= 0,
qr.hpp:15-18) of seeded Gaussians drawn from one RngStream (rng.cpp:72-79, U first,
then V); config 4 adds 1e-6 N(0,1) from substream 1. The QR and the product run in numpy
with OpenBLAS pinned to ONE thread and the Haswell kernels (OPENBLAS_CORETYPE), which is
what makes the bytes identical on this container and on any x86-64 GPU box host: the
golden fixtures under tests/golden/ record the SHA-256 of A, and the parity tests check
it before comparing results. OpenBLAS reads the pinning variables when it loads, so the
matrix is built in a child interpreter that sets them first.

Gaussians come from either this repo's host generator (libqbfac_matgen.so) or the
reference's own RngStream compiled into oracle/_ref (bench.py's reference arm, which must
not load this repo's libraries); the two streams are bit-identical
(tests/test_host.py), so both sources give the same A.

  python tools/pinned_inputs.py --cfg 2 --out A.npy [--gauss repo|oracle]
"""
from __future__ import annotations

import argparse
import hashlib
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PIN_ENV = {"OPENBLAS_CORETYPE": "Haswell", "OPENBLAS_NUM_THREADS": "1", "OMP_NUM_THREADS": "1",
           "MKL_NUM_THREADS": "1"}
CACHE = os.environ.get("QBFAC_INPUT_CACHE", os.path.join(ROOT, ".cache", "inputs"))

RECIPES = {
    "2": dict(m=8000, n=8000, seed=2, sigma="inv", noise=0.0),
    "4": dict(m=40000, n=20000, seed=4, sigma="exp60_r400", noise=1e-6),
    # small stand-ins of the same recipes (CPU tests of the generator itself)
    "2s": dict(m=600, n=600, seed=2, sigma="inv", noise=0.0),
    "4s": dict(m=900, n=700, seed=4, sigma="exp60_r400", noise=1e-6),
}


def _sigma(kind, n):
    import numpy as np
    j = np.arange(1, n + 1, dtype=np.float64)
    if kind == "inv":
        return 1.0 / j
    if kind == "exp60_r400":
        return np.exp(-np.arange(1, 401, dtype=np.float64) / 60.0)
    raise ValueError(kind)


def _build(cfg: str, out: str, gauss: str) -> str:
    """Runs in the pinned child: writes A (column-major .npy) and returns its SHA-256."""
    import numpy as np
    sys.path.insert(0, ROOT)
    if gauss == "oracle":
        from oracle import oracle as O

        def g(rows, cols, seed, stream, skip):
            return O.gaussian(rows, cols, seed, stream, skip)
    else:
        from paper_1606_09402_b200 import matgen

        def g(rows, cols, seed, stream, skip):
            return matgen.host_gaussian(rows, cols, seed, stream, skip)
    rc = RECIPES[str(cfg)]
    m, n, seed = rc["m"], rc["n"], rc["seed"]
    sig = _sigma(rc["sigma"], n)
    r = len(sig)

    def qpos(a):
        q, rr = np.linalg.qr(a)
        sg = np.sign(np.diag(rr))
        sg[sg == 0] = 1.0
        return q * sg

    u = qpos(g(m, r, seed, 0, 0))
    v = qpos(g(n, r, seed, 0, m * r))
    a = np.asfortranarray((u * sig) @ v.T)
    del u, v
    if rc["noise"]:
        if gauss == "oracle":
            a += rc["noise"] * g(m, n, seed, 1, 0)
        else:
            import ctypes as C
            matgen.mglib().qbm_gaussian_add(seed, 1, 0, m * n, rc["noise"], a.ctypes.data_as(C.c_void_p))
    np.save(out, a)
    return hashlib.sha256(memoryview(a.reshape(-1, order="F"))).hexdigest()


def matrix(cfg, gauss: str = "repo", expect_sha: str | None = None, cache: str | None = None):
    """A for config `cfg` as a read-only column-major memmap, built once per cache dir.
    Returns (A, sha256)."""
    import numpy as np
    cache = cache or CACHE
    os.makedirs(cache, exist_ok=True)
    path = os.path.join(cache, f"cfg{cfg}_A.npy")
    shap = path + ".sha256"
    if not (os.path.exists(path) and os.path.exists(shap)):
        env = dict(os.environ, **PIN_ENV)
        t0 = time.time()
        tmp = path + f".tmp{os.getpid()}.npy"
        subprocess.check_call([sys.executable, os.path.abspath(__file__), "--cfg", str(cfg), "--out", tmp,
                               "--gauss", gauss], env=env)
        os.replace(tmp, path)
        os.replace(tmp + ".sha256", shap)
        print(f"[pinned_inputs] cfg{cfg} A built in {time.time() - t0:.1f} s", file=sys.stderr)
    sha = open(shap).read().strip()
    a = np.load(path, mmap_mode="r")
    if expect_sha is not None and sha != expect_sha:
        raise AssertionError(f"cfg{cfg} A differs from the golden input: sha {sha[:16]} != {expect_sha[:16]}")
    return a, sha


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", required=True, choices=sorted(RECIPES))
    ap.add_argument("--out", required=True)
    ap.add_argument("--gauss", default="repo", choices=["repo", "oracle"])
    args = ap.parse_args()
    for k, v in PIN_ENV.items():
        if os.environ.get(k) != v:
            raise SystemExit(f"pinned_inputs: {k} must be {v} before numpy loads (use matrix())")
    sha = _build(args.cfg, args.out, args.gauss)
    with open(args.out + ".sha256", "w") as f:
        f.write(sha + "\n")


if __name__ == "__main__":
    main()

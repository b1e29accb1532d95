"""Full-size oracle runs of BASELINE configs 2, 4 and 5 (CPU: the reference's own kernels,
RNG and containers + the restated algorithm layer, oracle/_ref/libqbref.so). Writes
tests/golden/cfg{N}_full_{lane}.json: the input fingerprint, rank, passes, termination,
E, ||A||^2, sigma(B), the E trace and the explicit error ||A - QB||_F, plus the oracle's
own wall time. `--lane scalar` runs the reference's scalar kernel lane
(QBFAC_KERNELS=scalar, kernels_dispatch.cpp:38-50) to record the reference's own
lane-to-lane spread, the envelope the randQB_FP parity tests allow.

  python tools/oracle_full.py --cfg 2 [--lane avx2|scalar]

Config 2 takes ~3 min per lane on one core, config 4 ~5 min, config 5 ~1 h.
"""
import argparse
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

PARAMS = {
    2: dict(alg="fp", b=50, power=1, eps_rel=5e-2, l_budget=2000, max_rank=2000, seed=42,
            desc="cfg2 full: randQB_FP dense 8000x8000 sigma=1/j (pinned A, seed 2), b=50, P=1, eps=5e-2 rel, "
                 "l~=2000, Omega RngStream(42)"),
    4: dict(alg="single_pass", b=100, power=0, fixed_rank=(400, 0), seed=42,
            desc="cfg4 full: single-pass FP 40000x20000 rank-400 exp(-j/60) + 1e-6 noise (pinned A, seed 4), "
                 "l=400, b=100, Omega RngStream(42)"),
    5: dict(alg="ei", b=100, power=2, eps_rel=0.6, max_rank=2000, seed=42,
            desc="cfg5 full: randQB_EI CSR 2e6x5e5 Zipf(1.1) 2e8 nnz (seed 5), b=100, P=2, eps=0.6 rel, cap 2000, "
                 "Omega RngStream(42)"),
}


def csr_sha(csr):
    h = hashlib.sha256()
    for x in csr[2:]:
        h.update(memoryview(x))
    return h.hexdigest()


def csr_explicit_error(csr, q, b):
    """||A - QB||_F via ||A||^2 - 2<Q^T A, B> + <Q^T Q, B B^T> (no dense m x n)."""
    import numpy as np
    import scipy.sparse as sp
    m, n, rp, ci, v = csr
    a = sp.csr_matrix((v, ci, rp), shape=(m, n))
    qta = (a.T @ q).T  # k x n
    na = float(v @ v)
    val = na - 2.0 * float(np.sum(qta * b)) + float(np.sum((q.T @ q) * (b @ b.T)))
    return float(np.sqrt(max(val, 0.0)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, required=True, choices=[2, 4, 5])
    ap.add_argument("--lane", default="avx2", choices=["avx2", "scalar"])
    args = ap.parse_args()
    if args.lane == "scalar" and os.environ.get("QBFAC_KERNELS") != "scalar":
        os.environ["QBFAC_KERNELS"] = "scalar"
        os.execv(sys.executable, [sys.executable] + sys.argv)
    import numpy as np

    from oracle import oracle as O
    p = PARAMS[args.cfg]
    if args.cfg == 5:
        from paper_1606_09402_b200 import matgen
        csr = matgen.csr_zipf(2_000_000, 500_000, alpha=1.1, target_nnz=2e8, seed=5)
        a, fp = None, {"csr_sha256": csr_sha(csr), "nnz": int(len(csr[4]))}
        norm = float(np.sqrt(O.csr_frob_sq(csr)))
    else:
        import pinned_inputs
        a, sha = pinned_inputs.matrix(args.cfg)
        a = np.asfortranarray(a)
        csr, fp = None, {"a_sha256": sha}
        norm = float(np.linalg.norm(a))
    kw = dict(b=p["b"], power=p["power"], seed=p["seed"])
    if "fixed_rank" in p:
        kw["fixed_rank"] = p["fixed_rank"]
        eps = 0.0
    else:
        eps = p["eps_rel"] * norm
        kw.update(eps_abs=eps, max_rank=p["max_rank"])
    if "l_budget" in p:
        kw["l_budget"] = p["l_budget"]
    t0 = time.perf_counter()
    r = O.run(p["alg"], a=a, csr=csr, **kw)
    t = time.perf_counter() - t0
    assert O.lane_name() == args.lane, O.lane_name()
    s = np.linalg.svd(r.B, compute_uv=False) if r.rank else np.zeros(0)
    if csr is not None:
        xerr = csr_explicit_error(csr, r.Q, r.B)
    else:
        xerr = float(np.linalg.norm(a - r.Q @ r.B))
    loss = float(np.abs(r.Q.T @ r.Q - np.eye(r.rank)).sum(axis=1).max()) if r.rank else 0.0
    out = {"config": p["desc"], "lane": args.lane, **fp, "eps_abs": eps, "params": {k: v for k, v in kw.items()},
           "rank": r.rank, "passes": r.passes, "terminated_by": r.terminated_by, "E": r.E,
           "norm_a_sq": r.norm_a_sq, "sigma": s.tolist(), "e_trace": r.e_trace.tolist(),
           "explicit_error": xerr, "orth_loss": loss, "oracle_seconds": t, "cores": 1}
    path = os.path.join(ROOT, "tests", "golden", f"cfg{args.cfg}_full_{args.lane}.json")
    json.dump(out, open(path, "w"))
    print(f"cfg{args.cfg} {args.lane}: rank {r.rank} passes {r.passes} {r.terminated_by} E {r.E:.6e} "
          f"err {xerr:.6e} in {t:.1f} s -> {path}")


if __name__ == "__main__":
    main()

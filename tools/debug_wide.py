import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O
from paper_1606_09402_b200 import matgen, qbfac
ctx = qbfac.default_context()
a = matgen.synthesize(800, 700, matgen.spectrum("exp_decay", 700, tau=60.0), 17)
eps = 1e-4 * np.linalg.norm(a)
def sv(b): return np.linalg.svd(b, compute_uv=False)
for b in (100, 150):
    for alg, kw in (("fp", dict(power=1, eps_abs=eps, l_budget=450)), ("fp_fixed_rank", dict(fixed_rank=(300, 0), reorth=False)),
                    ("fp_fixed_rank", dict(fixed_rank=(300, 0), reorth=True))):
        ref = O.run(alg, a, b=b, seed=4, **kw)
        if alg == "fp":
            got = qbfac.rand_qb_fp(qbfac.MatrixHandle.dense(a, ctx), eps, b, 1, 450, qbfac.RngStream(4))
        else:
            got = qbfac.rand_qb_fp_fixed_rank(qbfac.MatrixHandle.dense(a, ctx), 300, 0, b, kw["reorth"], qbfac.RngStream(4))
        n = min(got.rank, ref.rank)
        s1, s2 = sv(got.B)[:n], sv(ref.B)[:n]
        rel = np.abs(s1 - s2) / s2
        bq = np.linalg.norm(got.B - got.Q.T @ a) / np.linalg.norm(a)
        bqr = np.linalg.norm(ref.B - ref.Q.T @ a) / np.linalg.norm(a)
        oq = np.abs(got.Q.T @ got.Q - np.eye(got.rank)).max()
        print(f"b={b} {alg} {kw.get('reorth','')}: rank {got.rank}/{ref.rank} passes {got.passes}/{ref.passes} "
              f"sig rel max {rel.max():.2e} first {rel[:3]} | B-QtA gpu {bq:.2e} ref {bqr:.2e} | orth {oq:.1e}", flush=True)

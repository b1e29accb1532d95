"""Regenerate tests/golden/*.json from the oracle (reference kernels + restated
algorithm layer). Run in the container that has /root/reference (oracle/_ref built).

  python tools/make_golden.py
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_1606_09402_b200 import matgen  # noqa: E402


def summary(r, a=None, csr=None, **extra):
    s = np.linalg.svd(r.B, compute_uv=False) if r.rank else np.zeros(0)
    d = {"rank": r.rank, "passes": r.passes, "E": r.E, "norm_a_sq": r.norm_a_sq, "terminated_by": r.terminated_by,
         "sigma_top": s[:20].tolist(), "sigma_tail": s[-5:].tolist(), "e_trace": r.e_trace.tolist(),
         "explicit_error": O.explicit_error(r.Q, r.B, a=a, csr=csr) if r.rank else None, "lane": O.lane_name()}
    d.update(extra)
    return d


def main():
    out = os.path.join(ROOT, "tests", "golden")
    os.makedirs(out, exist_ok=True)
    a = matgen.cfg1_matrix()
    eps = 1e-2 * float(np.linalg.norm(a))
    r = O.run("ei", a, b=20, power=0, eps_abs=eps, max_rank=1000, seed=42)
    json.dump(summary(r, a=a, eps_abs=eps, config="cfg1: EI dense 2000x2000, b=20, P=0, eps=1e-2 rel, cap 1000, "
                                                   "A seed 1, Omega RngStream(42)"),
              open(os.path.join(out, "cfg1_ei.json"), "w"), indent=1)
    csr = matgen.csr_uniform(3000, 1500, 20, seed=3000)
    eps = 0.5 * float(np.sqrt(O.csr_frob_sq(csr)))
    r = O.run("ei", csr=csr, b=20, power=1, eps_abs=eps, max_rank=200, seed=42)
    json.dump(summary(r, csr=csr, eps_abs=eps, config="cfg3 recipe at 3000x1500, 20/row, EI b=20 P=1 eps=0.5 rel cap 200"),
              open(os.path.join(out, "cfg3_small_ei.json"), "w"), indent=1)
    a = matgen.synthesize(400, 400, matgen.spectrum("inv", 400), 11)
    eps = 1e-2 * float(np.linalg.norm(a))
    r = O.run("fp", a, b=10, power=1, eps_abs=eps, l_budget=200, seed=6)
    json.dump(summary(r, a=a, eps_abs=eps, config="cfg2 recipe at 400x400 (sigma=1/j, seed 11), FP b=10 P=1 "
                                                   "eps=1e-2 rel l=200"),
              open(os.path.join(out, "cfg2_small_fp.json"), "w"), indent=1)
    print("golden written to", out)


if __name__ == "__main__":
    main()

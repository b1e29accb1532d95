"""ORACLE — TEST INFRASTRUCTURE ONLY.

Runs the oracle with the reference's SCALAR kernel lane (QBFAC_KERNELS=scalar,
/root/reference/proj/src/kernels_dispatch.cpp:38-50) in a child process. The
reference states that lanes "may reassociate reductions, so results can differ
between lanes by O(eps) rounding noise" (kernels.hpp:10-11); the scalar-vs-AVX2
spread of a factorization is therefore the reference's own reproducibility
floor, used by the parity tests for randQB_FP, whose B_i update amplifies
rounding (PAPER.md Remark 4.1).
"""
from __future__ import annotations

import os
import pickle
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)

_CHILD = r"""
import pickle, sys
sys.path.insert(0, {root!r})
from oracle import oracle as O
args, kw = pickle.load(open({inp!r}, "rb"))
r = O.run(*args, **kw)
assert O.lane_name() == "scalar", O.lane_name()
pickle.dump(r, open({out!r}, "wb"))
"""


def run_scalar(*args, **kw):
    with tempfile.TemporaryDirectory() as d:
        inp, out = os.path.join(d, "in.pkl"), os.path.join(d, "out.pkl")
        pickle.dump((args, kw), open(inp, "wb"))
        env = dict(os.environ, QBFAC_KERNELS="scalar")
        subprocess.check_call([sys.executable, "-c", _CHILD.format(root=ROOT, inp=inp, out=out)], env=env)
        return pickle.load(open(out, "rb"))

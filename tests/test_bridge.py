"""The reference-side C++ binding (include/qbfac/qb_gpu.hpp) used as a drop-in:
reference MatrixHandle / RngStream objects factorized by the restated CPU algorithm
and by qbfac::gpu::* in the same process (oracle/bridge_demo.cpp)."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEMO = os.path.join(ROOT, "oracle", "_ref", "bridge_demo")


@pytest.mark.gpu
def test_reference_binding_drop_in():
    if not os.path.exists(DEMO):
        pytest.skip("bridge_demo not built (needs /root/reference at build time)")
    out = subprocess.run([DEMO], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    cases = {d["case"]: d for d in (json.loads(l) for l in out.stdout.splitlines() if l.startswith("{"))}
    for name in ("ei_dense_300", "fp_dense_400", "ei_csr_2000x1500"):
        c = cases[name]
        assert c["rank_cpu"] == c["rank_gpu"], c
        assert c["term_cpu"] == c["term_gpu"], c
        assert c["passes_cpu"] == c["passes_gpu"], c          # PassCounter advanced identically
        assert c["rng_next_cpu"] == c["rng_next_gpu"], c      # RngStream left in the same state
        assert abs(c["err_cpu"] - c["err_gpu"]) <= 1e-8 * c["err_cpu"], c
    assert cases["floor"]["thrown"] is True
    for draws in (1, 2):  # a consumed RngStream is rejected before any device work
        c = cases[f"consumed_rng_{draws}"]
        assert c["thrown"] is True and c["passes"] == 0, c


def test_binding_header_compiles_against_reference_headers():
    """Host-only check: the binding header compiles with the reference's include tree."""
    ref = "/root/reference/proj/include"
    if not os.path.isdir(ref):
        pytest.skip("reference headers absent")
    src = '#include "qbfac/qb_gpu.hpp"\nint main(){return 0;}\n'
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-x", "c++", "-", f"-I{ref}",
                        f"-I{ROOT}/oracle/shim", f"-I{ROOT}/include"], input=src, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr

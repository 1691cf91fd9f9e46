"""Parity against committed golden vectors produced by the reference itself
(tests/golden/make_golden.py runs oracle/_ref, the unmodified reference
headers compiled in place).  The CPU half checks the oracle; the GPU half
checks the CUDA path with the project's bar (aggregation, level sizes / nnz /
operator complexity and coarse values bitwise; iterations +-1; u within 1e-12)."""
import os

import numpy as np
import pytest

import bindings as ob
from paper_1209_5421_b200 import problems

G = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden.npz"))
CASES = {
    "poisson5_40": lambda: problems.poisson5(40),
    "jitter_48": lambda: problems.jittered_p1(48),
    "graded_64": lambda: problems.graded_p1(64, 1.3),
    "disk_40": lambda: problems.disk_p1(40),
    "jump_48": lambda: problems.jittered_p1(48, jump=1e3),
}


def _check_setup(name, e):
    assert np.array_equal(e["levels"][0]["agg_of"], G[f"{name}/agg_of"])
    assert np.array_equal(np.array(e["stats"]["sizes"], np.int64), G[f"{name}/sizes"])
    assert np.array_equal(np.array(e["stats"]["nnz"], np.int64), G[f"{name}/nnz"])
    assert e["stats"]["operator_complexity"] == G[f"{name}/opcx"][0]
    assert np.array_equal(e["levels"][1]["ell_val"], G[f"{name}/ell_val_L"])
    assert np.array_equal(e["coarsest_lu"], G[f"{name}/coarsest_lu"])


@pytest.mark.parametrize("name", list(CASES))
def test_oracle_matches_golden(name):
    s = CASES[name]()
    h = ob.CpuHierarchy("oracle", s.A, s.coords)
    _check_setup(name, h.export())
    r = h.solve(s.b)
    assert r["iterations"] == G[f"{name}/iterations"][0]
    assert np.array_equal(r["residual_history"], G[f"{name}/residual_history"])
    assert np.array_equal(r["u"], G[f"{name}/u"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(CASES))
def test_gpu_matches_golden(gpu_api, name):
    s = CASES[name]()
    h = gpu_api.setup_hierarchy(s.A, s.coords)
    _check_setup(name, h.export())
    r = gpu_api.solve(s.A, s.b, h)
    assert abs(r.iterations - G[f"{name}/iterations"][0]) <= 1
    ug = G[f"{name}/u"]
    assert np.max(np.abs(r.u - ug)) / np.max(np.abs(ug)) <= 1e-12

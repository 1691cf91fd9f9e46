"""BASELINE.json full-size configurations on the GPU against the reference
itself (oracle/_ref: the unmodified reference headers compiled in place, run
with every host thread -- its results are bitwise independent of the thread
count, parallel.hpp:1-9), on inputs byte-identical to the reference's own
generators (tests/test_generators.py):

  C1 jittered P1 n=1025, C2 graded_mesh(2049,1.3), C3 jittered P1 n=4097,
  C4 jump 1e3 on the C3 mesh, C5 5-point n=4097 (the weak-scaling base).

Per configuration: every exported hierarchy field bitwise (aggregation maps,
member lists, active flags, colourings, every level's stencil pattern and
values, block and coarsest LU factors, statistics / operator complexity),
iterations within +-1 of the reference (and of SURVEY 8(c)'s goldens),
||u - u_ref||_inf / ||u_ref||_inf <= 1e-12, and the true residual recomputed
on the host meets rtol."""
import os

import numpy as np
import pytest
import scipy.sparse as sp

import bindings as ob
from paper_1209_5421_b200 import problems
from test_gpu_parity import compare_exports

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(900)]

U_TOL = 1e-12


def _true_rel_residual(s, u):
    A = sp.csr_matrix((s.A.values, s.A.col_idx, s.A.row_ptr), shape=(s.A.n_rows, s.A.n_rows))
    return np.linalg.norm(s.b - A @ u) / np.linalg.norm(s.b)


# name: (generator, SURVEY 8(c) golden iterations, golden operator complexity)
FULL = {
    "C1_jitter_1025": (lambda: problems.jittered_p1(1025), 12, 1.4274),
    "C2_graded_2049": (lambda: problems.graded_p1(2049, 1.3), 25, 1.4280),
    "C3_jitter_4097": (lambda: problems.jittered_p1(4097), 13, 1.4283),
    "C4_jump1e3_4097": (lambda: problems.jittered_p1(4097, jump=1e3), 34, None),
    "C5_poisson5_4097": (lambda: problems.poisson5(4097), 12, 1.5995),
}


@pytest.mark.skipif(not ob.available("ref"), reason="oracle/_ref not built")
@pytest.mark.parametrize("name", list(FULL))
def test_full_size_reference_parity(gpu_api, name):
    make, golden_iters, golden_opcx = FULL[name]
    s = make()
    ob.set_ref_threads(os.cpu_count() or 1)
    ref = ob.CpuHierarchy("ref", s.A, s.coords)
    rr = ref.solve(s.b)
    h = gpu_api.setup_hierarchy(s.A, s.coords)
    r = gpu_api.solve(s.A, s.b, h)
    # setup: every exported field bitwise
    eo = ref.export()
    del ref
    eg = h.export()
    compare_exports(eg, eo, exact_values=True)
    if golden_opcx is not None:
        assert round(eg["stats"]["operator_complexity"], 4) == golden_opcx
    del eg, eo
    # solve
    assert r.converged and rr["converged"]
    assert abs(r.iterations - rr["iterations"]) <= 1, (r.iterations, rr["iterations"])
    assert abs(rr["iterations"] - golden_iters) <= 1, rr["iterations"]
    err = np.max(np.abs(r.u - rr["u"])) / np.max(np.abs(rr["u"]))
    assert err <= U_TOL, err
    assert _true_rel_residual(s, r.u) <= 1.0e-6 * (1 + 1e-9)
    print(f"{name}: N={s.A.n_rows} iterations gpu={r.iterations} ref={rr['iterations']} max rel du={err:.2e}")


def test_full_size_modes_agree():
    from paper_1209_5421_b200 import api
    s = problems.jittered_p1(1025)
    us = []
    for bs in (0, 1):
        h = api.setup_hierarchy(s.A, s.coords, gpu=api.GpuOptions(block_solve=bs, coarse_solve=bs))
        r = api.solve(s.A, s.b, h)
        us.append((r.iterations, r.u))
    assert us[0][0] == us[1][0]
    assert np.max(np.abs(us[0][1] - us[1][1])) / np.max(np.abs(us[1][1])) <= 1e-12


@pytest.mark.parametrize("opts", [dict(cluster_tier=False), dict(fused_max_cells=256), dict(fused_max_cells=64),
                                  dict(use_graphs=False)])
def test_full_size_tiers_agree(opts):
    """C1 at full size through every coarse-tier configuration: the cluster
    tier off, the single-CTA tier cut to 256 / 64 cells (more levels on the TMA
    tile kernels), eager launches -- same iterations, solutions within the
    parity tolerance of the default path."""
    from paper_1209_5421_b200 import api
    s = problems.jittered_p1(1025)
    ref = api.solve(s.A, s.b, api.setup_hierarchy(s.A, s.coords))
    r = api.solve(s.A, s.b, api.setup_hierarchy(s.A, s.coords, gpu=api.GpuOptions(**opts)))
    assert r.iterations == ref.iterations
    assert np.max(np.abs(r.u - ref.u)) / np.max(np.abs(ref.u)) <= 1e-12

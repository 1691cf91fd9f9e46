"""The 128x128-cell level as one 16-CTA thread-block cluster per visit half
(csrc/cluster16.cu): oracle parity (iterations +-1, u within 1e-12),
agreement with the overlapped-tile path (same smoothed values; only the
inner-product tree differs), fewer launches than the tile path (so the
cluster kernels are the ones that ran), and determinism."""
import numpy as np
import pytest

import bindings as ob
from paper_1209_5421_b200 import problems

pytestmark = pytest.mark.gpu

U_TOL = 1e-12

CASES = {
    "jitter_257": lambda: problems.jittered_p1(257),
    "graded_257": lambda: problems.graded_p1(257, 1.3),
    "poisson5_257": lambda: problems.poisson5(257),
    "jump_257": lambda: problems.jittered_p1(257, jump=1e3),
    "disk_300": lambda: problems.disk_p1(300),
}


def _rel(a, b):
    return np.max(np.abs(a - b)) / np.max(np.abs(b))


def _run(gpu_api, s, g, co):
    h = gpu_api.setup_hierarchy(s.A, s.coords, gpu=g)
    r1 = gpu_api.solve(s.A, s.b, h, co)
    n0 = gpu_api.launch_count()
    r2 = gpu_api.solve(s.A, s.b, h, co)
    return r1, r2, gpu_api.launch_count() - n0


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("opts", [dict(), dict(n_inner=1), dict(n_inner=3), dict(pre_sweeps=2, post_sweeps=2),
                                  dict(pre_sweeps=2, post_sweeps=1), dict(max_directions=2)])
def test_cluster16_matches_oracle_and_tiles(gpu_api, name, opts):
    s = CASES[name]()
    co = gpu_api.CycleOptions(**opts)
    on, on2, n_on = _run(gpu_api, s, gpu_api.GpuOptions(cluster16=True), co)
    off, _, n_off = _run(gpu_api, s, gpu_api.GpuOptions(cluster16=False), co)
    ref = ob.CpuHierarchy("oracle", s.A, s.coords).solve(s.b, ob.cycle_opts(**opts))
    assert abs(on.iterations - ref["iterations"]) <= 1
    assert _rel(on.u, ref["u"]) <= U_TOL
    assert on.iterations == off.iterations
    assert _rel(on.u, off.u) <= U_TOL
    assert np.array_equal(on.u, on2.u)   # deterministic
    # the cluster up kernel absorbs the A-orthogonalisation launches of steps >= 1
    if co.n_inner >= 2:
        assert n_on < n_off, (n_on, n_off)
    else:
        assert n_on == n_off, (n_on, n_off)


def test_cluster16_graphs_off_and_lu_coarse(gpu_api):
    s = problems.jittered_p1(257)
    ref = ob.CpuHierarchy("oracle", s.A, s.coords).solve(s.b)
    for g in (gpu_api.GpuOptions(use_graphs=False), gpu_api.GpuOptions(coarse_solve=1),
              gpu_api.GpuOptions(cluster_tier=False, fused_max_cells=256)):
        r = gpu_api.solve(s.A, s.b, gpu_api.setup_hierarchy(s.A, s.coords, gpu=g))
        assert abs(r.iterations - ref["iterations"]) <= 1
        assert _rel(r.u, ref["u"]) <= U_TOL

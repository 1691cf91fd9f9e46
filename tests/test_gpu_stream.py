"""Row-wavefront kernels for the large structured levels (csrc/stream.cu),
forced onto small levels with GpuOptions.stream_min_width so every problem
family runs them: oracle parity (iterations +-1, u within 1e-12), agreement
with the overlapped-tile path (same smoothed values; only the inner-product
tree differs), determinism, and the multi-part (in-process) path where the
stream kernels cover each part's rectangle."""
import numpy as np
import pytest

import bindings as ob
from paper_1209_5421_b200 import problems

pytestmark = pytest.mark.gpu

U_TOL = 1e-12

CASES = {
    "jitter_129": lambda: problems.jittered_p1(129),
    "graded_129": lambda: problems.graded_p1(129, 1.3),
    "disk_96": lambda: problems.disk_p1(96),
    "poisson5_257": lambda: problems.poisson5(257),
    "jump_129": lambda: problems.jittered_p1(129, jump=1e3),
    "graded2_96": lambda: problems.graded_p1(96, 2.0),
}


def _rel(a, b):
    return np.max(np.abs(a - b)) / np.max(np.abs(b))


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("smw", [16, 32])
def test_stream_matches_oracle_and_tiles(gpu_api, name, smw):
    s = CASES[name]()
    tiles = gpu_api.GpuOptions(stream_min_width=-1, block_solve=1 if name == "graded2_96" else 0)
    strm = gpu_api.GpuOptions(stream_min_width=smw, block_solve=tiles.block_solve)
    rt = gpu_api.solve(s.A, s.b, gpu_api.setup_hierarchy(s.A, s.coords, gpu=tiles))
    h = gpu_api.setup_hierarchy(s.A, s.coords, gpu=strm)
    rs = gpu_api.solve(s.A, s.b, h)
    rs2 = gpu_api.solve(s.A, s.b, h)
    ref = ob.CpuHierarchy("oracle", s.A, s.coords).solve(s.b)
    assert abs(rs.iterations - ref["iterations"]) <= 1
    assert _rel(rs.u, ref["u"]) <= U_TOL
    assert rs.iterations == rt.iterations
    assert _rel(rs.u, rt.u) <= U_TOL
    assert np.array_equal(rs.u, rs2.u)   # run-to-run bitwise


@pytest.mark.parametrize("opts", [dict(n_inner=1), dict(n_inner=3), dict(max_directions=2)])
def test_stream_cycle_options(gpu_api, opts):
    s = problems.jittered_p1(129)
    co = gpu_api.CycleOptions(**opts)
    r = gpu_api.solve(s.A, s.b, gpu_api.setup_hierarchy(s.A, s.coords, gpu=gpu_api.GpuOptions(stream_min_width=16)), co)
    ref = ob.CpuHierarchy("oracle", s.A, s.coords).solve(s.b, ob.cycle_opts(**opts))
    assert abs(r.iterations - ref["iterations"]) <= 1
    assert _rel(r.u, ref["u"]) <= U_TOL


@pytest.mark.parametrize("parts", [2, 4, 8])
def test_stream_parts(gpu_api, parts, monkeypatch):
    """Each part runs the stream kernels over its rectangle (halo from the ring exchange)."""
    monkeypatch.setenv("AUX_DIST_AGG_SIDE", "0")
    s = problems.jittered_p1(257)
    u, res, _ = gpu_api.solve_parts(s.A, s.coords, s.b, parts, gpu=gpu_api.GpuOptions(stream_min_width=32))
    ref = ob.CpuHierarchy("oracle", s.A, s.coords).solve(s.b)
    assert abs(res[0].iterations - ref["iterations"]) <= 1
    assert _rel(u, ref["u"]) <= U_TOL


def test_stream_default_on_c1(gpu_api):
    """C1 (n = 1025): level L is 512 cells wide, so the default width (1024) keeps
    the tiles; forcing 512 streams level L.  Same iterations, u within 1e-12."""
    s = problems.jittered_p1(1025)
    r0 = gpu_api.solve(s.A, s.b, gpu_api.setup_hierarchy(s.A, s.coords, gpu=gpu_api.GpuOptions(stream_min_width=-1)))
    r1 = gpu_api.solve(s.A, s.b, gpu_api.setup_hierarchy(s.A, s.coords, gpu=gpu_api.GpuOptions(stream_min_width=512)))
    assert r0.iterations == r1.iterations == 12
    assert _rel(r1.u, r0.u) <= U_TOL

"""CPU tests: pin the oracle (C restatement) to the reference itself
(oracle/_ref, the unmodified reference headers compiled in place) and to the
reference's own known-answer tests.  No GPU needed."""
import numpy as np
import pytest

import bindings as ob
from paper_1209_5421_b200 import problems

needs_ref = pytest.mark.skipif(not ob.available("ref"), reason="oracle/_ref not built (no /root/reference here)")


def _cmp(ea, eb):
    assert ea["box"] == eb["box"] and ea["depth"] == eb["depth"]
    assert ea["locality"] == eb["locality"]
    assert ea["stats"] == eb["stats"]
    for la, lb in zip(ea["levels"], eb["levels"]):
        assert la.keys() == lb.keys()
        for k in la:
            if isinstance(la[k], np.ndarray):
                assert np.array_equal(la[k], lb[k]), k
            else:
                assert la[k] == lb[k], k
    assert np.array_equal(ea["coarsest_lu"], eb["coarsest_lu"])
    assert np.array_equal(ea["coarsest_perm"], eb["coarsest_perm"])


CASES = {
    "poisson5_33": lambda: problems.poisson5(33),
    "poisson5_65": lambda: problems.poisson5(65),
    "jitter_40": lambda: problems.jittered_p1(40),
    "graded_48": lambda: problems.graded_p1(48, 1.3),
    "disk_40": lambda: problems.disk_p1(40),
    "graded2_40": lambda: problems.graded_p1(40, 2.0),
    "jump_40": lambda: problems.jittered_p1(40, jump=1e3),
    "tiny_direct": lambda: problems.poisson5(6),
}


@needs_ref
@pytest.mark.parametrize("name", list(CASES))
def test_oracle_equals_reference_bitwise(name):
    s = CASES[name]()
    a = ob.CpuHierarchy("oracle", s.A, s.coords)
    b = ob.CpuHierarchy("ref", s.A, s.coords)
    _cmp(a.export(), b.export())
    ra, rb = a.solve(s.b), b.solve(s.b)
    assert ra["iterations"] == rb["iterations"]
    assert np.array_equal(ra["u"], rb["u"])
    assert np.array_equal(ra["residual_history"], rb["residual_history"])


@needs_ref
@pytest.mark.parametrize("opts", [dict(lump_locality=True), dict(coarsest_size=4), dict(coarsest_size=200)])
def test_oracle_setup_options(opts):
    s = problems.graded_p1(40, 2.0)
    a = ob.CpuHierarchy("oracle", s.A, s.coords, ob.setup_opts(**opts))
    b = ob.CpuHierarchy("ref", s.A, s.coords, ob.setup_opts(**opts))
    _cmp(a.export(), b.export())
    assert np.array_equal(a.solve(s.b)["u"], b.solve(s.b)["u"])


@needs_ref
@pytest.mark.parametrize("opts", [dict(n_inner=1), dict(n_inner=3), dict(max_directions=2),
                                  dict(pre_sweeps=2, post_sweeps=3), dict(max_outer=2)])
def test_oracle_cycle_options(opts):
    s = problems.jittered_p1(40)
    a = ob.CpuHierarchy("oracle", s.A, s.coords)
    b = ob.CpuHierarchy("ref", s.A, s.coords)
    ra, rb = a.solve(s.b, ob.cycle_opts(**opts)), b.solve(s.b, ob.cycle_opts(**opts))
    assert ra["iterations"] == rb["iterations"]
    assert np.array_equal(ra["u"], rb["u"])


@needs_ref
def test_oracle_error_classes():
    s = problems.poisson5(12)
    for kind in ("oracle", "ref"):
        with pytest.raises(ob._abi.SizeError):
            ob.CpuHierarchy(kind, s.A, s.coords[:-1])
        xy = s.coords.copy()
        xy[:, 0] = 0.25
        with pytest.raises(ob._abi.GeometryError):
            ob.CpuHierarchy(kind, s.A, xy)
        xy = s.coords.copy()
        xy[2, 1] = np.inf
        with pytest.raises(ob._abi.ArgumentError):
            ob.CpuHierarchy(kind, s.A, xy)
        h = ob.CpuHierarchy(kind, s.A, s.coords)
        with pytest.raises(ob._abi.ArgumentError):
            h.solve(s.b, ob.cycle_opts(rtol=0.0))


# ---- the reference's own known-answer tests, re-expressed (tests/test_*.cpp)

@pytest.mark.parametrize("kind", ["oracle", "ref"])
def test_choose_depth_kat(kind):
    if kind == "ref" and not ob.available("ref"):
        pytest.skip("no _ref")
    # test_auxgrid.cpp:29-38
    for n, d in [(1000, 4), (16, 1), (1 << 20, 9), (64, 2), (65, 3)]:
        assert ob.choose_depth(kind, n) == d
    with pytest.raises(ob._abi.ArgumentError):
        ob.choose_depth(kind, 3)


@pytest.mark.parametrize("kind", ["oracle", "ref"])
def test_subregion_clamp_kat(kind):
    if kind == "ref" and not ob.available("ref"):
        pytest.skip("no _ref")
    box = (0.0, 1.0, 0.0, 1.0)
    # test_auxgrid.cpp:40-65: upper boundary clamps into the last cell, lexicographic x-fastest
    assert ob.subregion_of_point(kind, 1.0, 1.0, box, 2) == 15
    assert ob.subregion_of_point(kind, 0.0, 0.0, box, 2) == 0
    assert ob.subregion_of_point(kind, 0.26, 0.0, box, 2) == 1
    assert ob.subregion_of_point(kind, 0.0, 0.26, box, 2) == 4
    assert ob.subregion_of_point(kind, 0.99, 0.74, box, 1) == 3
    with pytest.raises(ob._abi.GeometryError):
        ob.subregion_of_point(kind, 1.5, 0.5, box, 2)


def _sequential_gs(col, val, b, x, order, n):
    # oracles.hpp:89-115: plain Gauss-Seidel in an explicit row order
    x = x.copy()
    for i in order:
        s = b[i]
        for t in range(1, 9):
            j = col[t * n + i]
            if j >= 0:
                s -= val[t * n + i] * x[j]
        x[i] = s / val[i]
    return x


@pytest.mark.parametrize("kind", ["oracle", "ref"])
def test_colored_sweep_equals_sequential(kind):
    if kind == "ref" and not ob.available("ref"):
        pytest.skip("no _ref")
    # test_smoother.cpp:69-88
    k, n = 2, 16
    col, val = problems.random_stencil(k, 17)
    b = problems.random_vector(n, 18)
    x0 = problems.random_vector(n, 19)
    w = 1 << k
    color = [(i % w) % 2 + 2 * ((i // w) % 2) for i in range(n)]
    fwd = [i for c in range(4) for i in range(n) if color[i] == c]
    rev = [i for c in (3, 2, 1, 0) for i in range(n) if color[i] == c]
    assert np.array_equal(ob.point_gs_sweep_ell(kind, k, col, val, b, x0, 0), _sequential_gs(col, val, b, x0, fwd, n))
    assert np.array_equal(ob.point_gs_sweep_ell(kind, k, col, val, b, x0, 1), _sequential_gs(col, val, b, x0, rev, n))


def test_stencil_rows_kat():
    # test_hierarchy.cpp:48-63 via a 16-DoF lattice: exported level-2 ELL columns
    s = problems.poisson5(5)          # 16 DoFs on a cell-centred 4x4 lattice
    h = ob.CpuHierarchy("oracle", s.A, s.coords, ob.setup_opts(coarsest_size=4))
    e = h.export()
    lv = [l for l in e["levels"] if l["structured"] and l["k"] == 1][0]
    row0 = [lv["ell_col"][t * 4 + 0] for t in range(9)]
    assert row0 == [0, 1, 3, 2, -1, -1, -1, -1, -1]


def test_dot_matches_reference_tree():
    if not ob.available("ref"):
        pytest.skip("no _ref")
    a = problems.random_vector(5000, 3)
    b = problems.random_vector(5000, 4)
    assert ob.dot("oracle", a, b) == ob.dot("ref", a, b)


@pytest.mark.parametrize("kind", ["oracle", "ref"])
def test_level_stack_n17_kat(kind):
    if kind == "ref" and not ob.available("ref"):
        pytest.skip("no _ref")
    # test_hierarchy.cpp:249-308: poisson n=17 -> sizes {256,64,16,4} below the finest with coarsest 4
    s = problems.poisson5(17)
    h = ob.CpuHierarchy(kind, s.A, s.coords, ob.setup_opts(coarsest_size=4))
    e = h.export()
    assert e["stats"]["sizes"] == [256, 64, 16, 4]
    assert [lv["k"] for lv in e["levels"]] == [4, 3, 2, 1]
    assert [lv["structured"] for lv in e["levels"]] == [False, True, True, True]
    assert e["depth"] == 3
    assert int(e["levels"][0]["block_size"].sum()) == 256
    assert 1.0 <= e["stats"]["operator_complexity"] < 2.0
    # test_hierarchy.cpp:310-317: default coarsest size stops at 64 cells
    s16 = problems.poisson5(16)
    e16 = ob.CpuHierarchy(kind, s16.A, s16.coords).export()
    assert e16["stats"]["sizes"] == [225, 64] and e16["levels"][1]["k"] == 3


def test_galerkin_dense_oracle_pinned_to_reference():
    """galerkin_dense (hierarchy.hpp:239-247) on random SPD matrices with random
    surjective partitions (acceptance.cpp:55-65) and on a level-L partition:
    oracle == reference bitwise."""
    from paper_1209_5421_b200 import problems
    rng = np.random.default_rng(5)
    cases = []
    for trial in range(6):
        n = 16 + 37 * trial
        A = problems.random_spd(n, 1000 + trial)
        n_agg = 4 + trial % 13
        agg = rng.integers(0, n_agg, n).astype(np.int32)
        agg[:n_agg] = np.arange(n_agg)   # surjective
        cases.append((A, agg, n_agg))
    s = problems.jittered_p1(33)
    e = ob.CpuHierarchy("ref", s.A, s.coords).export()
    cases.append((s.A, e["levels"][0]["agg_of"].astype(np.int32), int(e["levels"][1]["n"])))
    for A, agg, n_agg in cases:
        c_ref = ob.galerkin_dense("ref", A, agg, n_agg)
        c_orc = ob.galerkin_dense("oracle", A, agg, n_agg)
        assert np.array_equal(c_ref, c_orc)

"""The harness input generator (paper_1209_5421_b200/csrc/problems.cpp ->
libauxgen.so) against the reference's own generators, compiled in place from
/root/reference through oracle/ref_shim.cpp (oracle/_ref/libauxamg_ref.so):

  gen_poisson_uniform2d              problems.hpp:41-76
  structured_split_mesh + assemble   problems.hpp:80-105, 152-193 (csr_from_triplets sparse.hpp:193-215)
  testgen::graded_mesh / disk_mesh   tests/testgen.hpp:91-98, 132-158
  testgen::random_spd / random_stencil / random_vector   tests/testgen.hpp:18-86
  jitter (C1/C3) and jump coefficient (C4): SURVEY.md 8(d), restated in the shim
  around the reference's element_geometry + csr_from_triplets

Every array must be byte-identical, so every bench and parity input is
provably the reference's input.  The 16M-DoF sizes (C3/C4/C5) take ~30 s per
generator on one core and run in the GPU suite (tests/test_gpu_fullsize.py)."""
import numpy as np
import pytest

import bindings as ob
from paper_1209_5421_b200 import problems

pytestmark = pytest.mark.skipif(not ob.available("ref"), reason="oracle/_ref not built")


def same_system(a, b):
    assert a.A.n_rows == b.A.n_rows and a.A.nnz == b.A.nnz
    assert a.A.row_ptr.tobytes() == b.A.row_ptr.tobytes()
    assert a.A.col_idx.tobytes() == b.A.col_idx.tobytes()
    assert a.A.values.tobytes() == b.A.values.tobytes()
    assert a.b.tobytes() == b.b.tobytes()
    assert a.coords.tobytes() == b.coords.tobytes()


@pytest.mark.parametrize("kind,n,param,jump", [
    (0, 2, 0.0, 0.0), (0, 33, 0.0, 0.0), (0, 64, 0.0, 0.0),
    (1, 1, 0.0, 0.0), (1, 17, 0.0, 0.0), (1, 40, 0.0, 1e3),
    (2, 33, 0.15, 0.0), (2, 64, 0.15, 0.0), (2, 65, 0.15, 1e3), (2, 48, 0.15, 1e6),
    (3, 33, 1.3, 0.0), (3, 65, 2.0, 0.0), (3, 64, 1.3, 1e3),
    (4, 40, 0.48, 0.0), (4, 61, 0.3, 0.0), (4, 50, 0.48, 1e3),
])
def test_small_systems_and_meshes_identical(kind, n, param, jump):
    s, m = problems.make_with_mesh(kind, n, param, 1, jump) if kind else (problems.make(kind, n), None)
    if kind:
        r, rm = ob.ref_make(kind, n, param, 1, jump, mesh=True)
        assert m.nodes.tobytes() == rm.nodes.tobytes()
        assert np.array_equal(m.triangles, rm.triangles)
        assert np.array_equal(m.boundary, rm.boundary)
    else:
        r = ob.ref_make(kind, n)
    same_system(s, r)


def test_seeds_differ_and_match():
    for seed in (1, 2, 7):
        same_system(problems.jittered_p1(40, 0.15, seed), ob.ref_make(2, 40, 0.15, seed))


@pytest.mark.parametrize("name,kind,n,param,jump", [
    ("C1 jittered P1 n=1025", 2, 1025, 0.15, 0.0),
    ("C1 5-point companion n=1025", 0, 1025, 0.0, 0.0),
    ("C4 family jump 1e3 n=1025", 2, 1025, 0.15, 1e3),
    ("C2 graded_mesh(2049,1.3)", 3, 2049, 1.3, 0.0),
])
def test_baseline_sizes_identical(name, kind, n, param, jump):
    same_system(problems.make(kind, n, param, 1, jump), ob.ref_make(kind, n, param, 1, jump))


def test_random_generators_identical():
    for n, seed in ((3, 1), (12, 5), (40, 9)):
        a, b = problems.random_spd(n, seed), ob.ref_random_spd(n, seed)
        assert a.row_ptr.tobytes() == b.row_ptr.tobytes() and a.col_idx.tobytes() == b.col_idx.tobytes()
        assert a.values.tobytes() == b.values.tobytes()
    for k, seed in ((1, 3), (4, 11), (6, 2)):
        (c1, v1), (c2, v2) = problems.random_stencil(k, seed), ob.ref_random_stencil(k, seed)
        assert np.array_equal(c1, c2) and v1.tobytes() == v2.tobytes()
    assert problems.random_vector(1000, 4).tobytes() == ob.ref_random_vector(1000, 4).tobytes()
    assert problems.random_vector(77, 9, 0.1, 2.0).tobytes() == ob.ref_random_vector(77, 9, 0.1, 2.0).tobytes()

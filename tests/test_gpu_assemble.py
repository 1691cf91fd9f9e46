"""Device P1 FEM assembly: aux_assemble_p1 against the
reference's own assemble_fem_triangle + csr_from_triplets (problems.hpp:152-193,
sparse.hpp:193-215), compiled in place through oracle/ref_shim.cpp
(bindings.ref_make; the jump coefficient of C4 is the shim's restatement around
the reference's element_geometry).  Pattern, load vector,
coordinates and every entry summed from <= 2 contributions are bitwise; a
diagonal sums ~6 contributions, added in element order here and in the
reference's (unstable) std::sort order there, so it may differ in the last
bits.  The assembled system then runs setup + solve without leaving the GPU."""
import numpy as np
import pytest

import bindings as ob
from paper_1209_5421_b200 import problems

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind,n,param,jump", [
    (1, 33, 0.0, 0.0),          # structured split mesh
    (2, 64, 0.15, 0.0),         # jittered (C1/C3 family)
    (3, 65, 1.3, 0.0),          # graded (C2 family)
    (4, 40, 0.48, 0.0),         # disk: detected boundary
    (2, 48, 0.15, 1e3),         # jump coefficient (C4 family)
])
def test_assembly_matches_reference(gpu_api, kind, n, param, jump):
    s, m = ob.ref_make(kind, n, param, 1, jump, mesh=True)
    ds = gpu_api.DeviceSystem(m.nodes, m.triangles, m.boundary, 1.0, jump)
    A, b, xy = ds.to_host()
    assert A.n_rows == s.A.n_rows and A.nnz == s.A.nnz
    assert np.array_equal(A.row_ptr, s.A.row_ptr)
    assert np.array_equal(A.col_idx, s.A.col_idx)
    assert np.array_equal(b, s.b)
    assert np.array_equal(xy, s.coords)
    rows = np.repeat(np.arange(A.n_rows), np.diff(A.row_ptr))
    off = rows != A.col_idx
    assert np.array_equal(A.values[off], s.A.values[off])
    d = ~off
    rel = np.abs(A.values[d] - s.A.values[d]) / np.abs(s.A.values[d])
    assert rel.max() <= 2e-15, rel.max()   # <= 8 ulp: 6 terms summed in another order


def test_assembled_system_solves_on_device(gpu_api):
    import torch
    s, m = problems.make_with_mesh(2, 257, 0.15)
    ds = gpu_api.DeviceSystem(m.nodes, m.triangles, m.boundary)
    h = ds.setup()
    _, b_ptr, _ = ds.device_view()
    u = torch.empty(ds.n, dtype=torch.float64, device="cuda")
    r = gpu_api.solve_device(h, b_ptr, u.data_ptr(), ds.n)
    ref = gpu_api.solve(s.A, s.b, gpu_api.setup_hierarchy(s.A, s.coords))
    assert abs(r.iterations - ref.iterations) <= 1
    uu = u.cpu().numpy()
    assert np.max(np.abs(uu - ref.u)) / np.max(np.abs(ref.u)) <= 1e-12


def test_assembly_errors(gpu_api):
    s, m = problems.make_with_mesh(1, 9)
    bad = m.triangles.copy()
    bad[3, 1] = m.nodes.shape[0]
    with pytest.raises(gpu_api.ArgumentError):
        gpu_api.DeviceSystem(m.nodes, bad, m.boundary)
    deg = m.triangles.copy()
    deg[5] = [deg[5][0], deg[5][0], deg[5][1]]
    with pytest.raises(gpu_api.GeometryError, match="triangle 5"):
        gpu_api.DeviceSystem(m.nodes, deg, m.boundary)

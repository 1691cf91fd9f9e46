"""Drop-in boundary: solve(A, b, h) with an A other than the
setup matrix.  The reference runs the cycle on the hierarchy's copy of the
setup matrix and the outer A z on the caller's A (cycle.hpp:202-208, 228); the
B200 path reuses its device copy for the setup matrix and uploads any other
matrix for the outer product.  Compared with the reference itself (oracle/_ref)
on the same A: iterations +-1, u within 1e-12."""
import numpy as np
import pytest

import bindings as ob
from paper_1209_5421_b200 import problems

pytestmark = pytest.mark.gpu


def _check(gpu_api, s, A_solve, kind="ref"):
    h = gpu_api.setup_hierarchy(s.A, s.coords)
    r = gpu_api.solve(A_solve, s.b, h)
    ref = ob.CpuHierarchy(kind, s.A, s.coords)
    rr = ref.solve(s.b, A=A_solve)
    assert abs(r.iterations - rr["iterations"]) <= 1, (r.iterations, rr["iterations"])
    err = np.max(np.abs(r.u - rr["u"])) / np.max(np.abs(rr["u"]))
    assert err <= 1e-12, err
    return r


def _copy(A):
    return problems.CsrMatrix(A.n_rows, A.n_cols, A.row_ptr.copy(), A.col_idx.copy(), A.values.copy())


@pytest.mark.parametrize("maker", [lambda: problems.jittered_p1(64), lambda: problems.graded_p1(65, 1.3)])
def test_content_equal_copy(gpu_api, maker):
    s = maker()
    _check(gpu_api, s, _copy(s.A))


@pytest.mark.parametrize("maker", [lambda: problems.jittered_p1(64), lambda: problems.poisson5(60)])
def test_values_modified(gpu_api, maker):
    """Values changed symmetrically (a_ij *= 1 + 1e-3 ((i + j) mod 3)), so the
    caller's A stays SPD and the outer PCG converges on both sides; a
    non-symmetric edit makes the reference's own iteration chaotic under
    rounding (flexible PCG on a non-symmetric operator)."""
    s = maker()
    A2 = _copy(s.A)
    rows = np.repeat(np.arange(A2.n_rows), np.diff(A2.row_ptr))
    A2.values *= 1.0 + 1e-3 * ((rows + A2.col_idx) % 3)
    _check(gpu_api, s, A2)


def test_other_pattern_and_unsorted_columns(gpu_api):
    """An extra stored zero per row and reversed column order in every row: the
    reference's csr_spmv reads any CSR of the right order (sparse.hpp:141-150)."""
    s = problems.jittered_p1(48)
    A = s.A
    rows, cols, vals = [], [], []
    n = A.n_rows
    rp = [0]
    for r in range(n):
        c = list(A.col_idx[A.row_ptr[r]:A.row_ptr[r + 1]])
        v = list(A.values[A.row_ptr[r]:A.row_ptr[r + 1]] * 0.75)
        if (r + 3) % n not in c:
            c.append((r + 3) % n)
            v.append(0.0)
        cols += c[::-1]
        vals += v[::-1]
        rp.append(len(cols))
    A2 = problems.CsrMatrix(n, n, np.array(rp, np.int32), np.array(cols, np.int32), np.array(vals))
    _check(gpu_api, s, A2)


def test_setup_matrix_rescaled_in_place(gpu_api):
    """The setup matrix's own arrays rewritten after setup (as after a free and
    reallocation at the same addresses): the sampled fingerprint detects it."""
    s = problems.jittered_p1(64)
    A = _copy(s.A)
    h = gpu_api.setup_hierarchy(A, s.coords)
    ref = ob.CpuHierarchy("ref", _copy(A), s.coords)
    A.values *= 3.0
    r = gpu_api.solve(A, s.b, h)
    rr = ref.solve(s.b, A=A)
    assert abs(r.iterations - rr["iterations"]) <= 1
    assert np.max(np.abs(r.u - rr["u"])) / np.max(np.abs(rr["u"])) <= 1e-12


def test_wrong_order_and_bad_structure(gpu_api):
    s = problems.jittered_p1(32)
    h = gpu_api.setup_hierarchy(s.A, s.coords)
    t = problems.jittered_p1(31)
    with pytest.raises(gpu_api.SizeError):
        gpu_api.solve(t.A, t.b, h)
    A2 = _copy(s.A)
    A2.col_idx[5] = s.A.n_rows + 7
    with pytest.raises(gpu_api.StructureError, match="out of range"):
        gpu_api.solve(A2, s.b, h)

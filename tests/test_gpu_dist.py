"""Multi-GPU path on one B200: P parts of one distributed
hierarchy driven by P threads (CommLocal transport: the same kernels, ring
exchanges, ghost exchanges, all-reduces and part-0 agglomeration as the NCCL
path, with the transfers as device copies).  Checked against the oracle with
the single-GPU bar (iterations +-1, u within 1e-12) and against the one-part
hierarchy (global level sizes / nnz / operator complexity identical)."""
import numpy as np
import pytest

import bindings as ob
from paper_1209_5421_b200 import problems

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(600)]

U_TOL = 1e-12


@pytest.fixture(params=["512", "0"], ids=["agg512", "deep"])
def agg_side(request, monkeypatch):
    """Default agglomeration (levels of <= 512^2 cells on part 0) and the
    deepest distribution (every level with a tileable rectangle per part)."""
    monkeypatch.setenv("AUX_DIST_AGG_SIDE", request.param)
    return request.param


@pytest.mark.parametrize("parts", [1, 2, 4, 8])
@pytest.mark.parametrize("name,make", [
    ("jitter_257", lambda: problems.jittered_p1(257)),
    ("graded_257", lambda: problems.graded_p1(257, 1.3)),
    ("poisson5_300", lambda: problems.poisson5(300)),
])
def test_parts_match_oracle(gpu_api, parts, name, make, agg_side):
    s = make()
    u, res, st = gpu_api.solve_parts(s.A, s.coords, s.b, parts)
    ref = ob.CpuHierarchy("oracle", s.A, s.coords).solve(s.b)
    its = {r.iterations for r in res}
    assert len(its) == 1                      # every part ran the same outer loop
    assert abs(res[0].iterations - ref["iterations"]) <= 1
    err = np.max(np.abs(u - ref["u"])) / np.max(np.abs(ref["u"]))
    assert err <= U_TOL, err
    h1 = gpu_api.setup_hierarchy(s.A, s.coords)
    s1 = h1.stats()
    for sp in st:
        assert sp.levels == s1.levels and list(sp.sizes) == list(s1.sizes)
        assert list(sp.nnz) == list(s1.nnz)
        assert sp.operator_complexity == s1.operator_complexity


@pytest.mark.parametrize("parts", [2, 4, 8])
@pytest.mark.parametrize("name,make", [
    ("disk_257", lambda: problems.disk_p1(257)),                    # empty cells, curved boundary
    ("graded2_257", lambda: problems.graded_p1(257, 2.0)),          # dropped + same-colour couplings
    ("jump_257", lambda: problems.jittered_p1(257, jump=1e3)),      # jump coefficient (C4 family)
])
def test_parts_hard_problems(gpu_api, parts, name, make, agg_side):
    s = make()
    u, res, st = gpu_api.solve_parts(s.A, s.coords, s.b, parts)
    ref = ob.CpuHierarchy("oracle", s.A, s.coords).solve(s.b)
    assert abs(res[0].iterations - ref["iterations"]) <= 1
    err = np.max(np.abs(u - ref["u"])) / np.max(np.abs(ref["u"]))
    assert err <= U_TOL, err
    h1 = gpu_api.setup_hierarchy(s.A, s.coords)
    assert list(st[0].nnz) == list(h1.stats().nnz)
    assert h1.locality() == gpu_api.setup_hierarchy(s.A, s.coords).locality()


def test_parts_cycle_options(gpu_api):
    s = problems.jittered_p1(257)
    for o in (dict(pre_sweeps=2, post_sweeps=2), dict(n_inner=3), dict(max_directions=3)):
        u, res, _ = gpu_api.solve_parts(s.A, s.coords, s.b, 4, cycle=gpu_api.CycleOptions(**o))
        ref = ob.CpuHierarchy("oracle", s.A, s.coords).solve(s.b, ob.cycle_opts(**o))
        assert abs(res[0].iterations - ref["iterations"]) <= 1
        assert np.max(np.abs(u - ref["u"])) / np.max(np.abs(ref["u"])) <= U_TOL


def test_parts_errors_consistent(gpu_api):
    s = problems.poisson5(20)   # level-L grid too small for 8 parts
    with pytest.raises(gpu_api.ArgumentError):
        gpu_api.solve_parts(s.A, s.coords, s.b, 8)


def test_nccl_transport_single_rank(gpu_api):
    """The NCCL transport (dlopen'ed libnccl, shared communicator) with one rank:
    the code path a torchrun launch takes on every rank."""
    s = problems.jittered_p1(129)
    comm = gpu_api.NcclComm(gpu_api.nccl_unique_id(), 1, 0, 0)
    h = gpu_api.setup_hierarchy_dist(s.A, s.coords, 1, 0, comm=comm)
    r = gpu_api.solve(s.A, s.b, h)
    ref = ob.CpuHierarchy("oracle", s.A, s.coords).solve(s.b)
    assert abs(r.iterations - ref["iterations"]) <= 1
    assert np.max(np.abs(r.u - ref["u"])) / np.max(np.abs(ref["u"])) <= U_TOL
    assert sorted(gpu_api.part_dofs(h).tolist()) == list(range(s.A.n_rows))


@pytest.mark.parametrize("parts", [2, 4, 8])
def test_parts_partition_dofs(gpu_api, parts):
    """Every DoF is owned by exactly one part; parts own their rectangles' DoFs."""
    import threading
    s = problems.jittered_p1(257)
    grp = gpu_api.LocalGroup(parts)
    ids = [None] * parts

    def run(r):
        h = gpu_api.setup_hierarchy_dist(s.A, s.coords, parts, r, group=grp)
        ids[r] = gpu_api.part_dofs(h)
        del h

    th = [threading.Thread(target=run, args=(r,)) for r in range(parts)]
    [t.start() for t in th]
    [t.join() for t in th]
    allids = np.concatenate(ids)
    assert np.array_equal(np.sort(allids), np.arange(s.A.n_rows))
    assert max(len(i) for i in ids) < s.A.n_rows
    # the library's rows are exactly the host-side statement of the partition
    from paper_1209_5421_b200 import partition as pt
    P = pt.Partition(s.A, s.coords, parts)
    for r in range(parts):
        assert np.array_equal(ids[r], P.owned_dofs(r))


@pytest.mark.parametrize("parts", [4, 8])
def test_parts_full_size_c1(gpu_api, parts):
    """C1 (jittered P1, N = 1,048,576) split over 4 / 8 parts: SURVEY 8(c)
    golden iteration count (12) and the true residual."""
    import scipy.sparse as sp
    s = problems.jittered_p1(1025)
    u, res, st = gpu_api.solve_parts(s.A, s.coords, s.b, parts)
    assert res[0].converged and abs(res[0].iterations - 12) <= 1
    A = sp.csr_matrix((s.A.values, s.A.col_idx, s.A.row_ptr), shape=(s.A.n_rows, s.A.n_rows))
    assert np.linalg.norm(s.b - A @ u) / np.linalg.norm(s.b) <= 1e-6 * (1 + 1e-9)
    assert round(st[0].operator_complexity, 4) == 1.4274


def _corrupt_cases():
    s = problems.jittered_p1(129)
    n = s.A.n_rows
    cases = {}
    A = problems.CsrMatrix(n, n, s.A.row_ptr.copy(), s.A.col_idx.copy(), s.A.values.copy())
    r = n - 7   # a late row: owned by another part than the first one
    A.col_idx[A.row_ptr[r] + 1], A.col_idx[A.row_ptr[r]] = A.col_idx[A.row_ptr[r]], A.col_idx[A.row_ptr[r] + 1]
    cases["unsorted_row"] = (A, s.coords)
    A = problems.CsrMatrix(n, n, s.A.row_ptr.copy(), s.A.col_idx.copy(), s.A.values.copy())
    for r in (n // 3, 2 * n // 3):   # two bad diagonals in different parts: the lower row is reported
        p = A.row_ptr[r] + int(np.nonzero(A.col_idx[A.row_ptr[r]:A.row_ptr[r + 1]] == r)[0][0])
        A.values[p] = -1.0
    cases["bad_diagonals"] = (A, s.coords)
    A = problems.CsrMatrix(n, n, s.A.row_ptr.copy(), s.A.col_idx.copy(), s.A.values.copy())
    r = n // 2
    p = next(q for q in range(A.row_ptr[r], A.row_ptr[r + 1]) if A.col_idx[q] != r and A.values[q] != 0.0)
    A.values[p] *= 1.5   # one off-diagonal entry of a middle row (its transpose is untouched)
    cases["nonsymmetric"] = (A, s.coords)
    xy = s.coords.copy()
    xy[n - 3, 0] = np.nan
    cases["nan_coordinate"] = (s.A, xy)
    return cases, s.b


@pytest.mark.parametrize("parts", [2, 4])
def test_parts_errors_match_single_gpu(gpu_api, parts):
    """Validation over each part's own rows with all-reduced verdicts: every
    part raises exactly the error (class and message: lowest failing row) of
    the single-GPU setup, which matches the reference's."""
    cases, b = _corrupt_cases()
    for name, (A, xy) in cases.items():
        with pytest.raises(gpu_api.AuxamgError) as e1:
            gpu_api.setup_hierarchy(A, xy)
        with pytest.raises(gpu_api.AuxamgError) as ep:
            gpu_api.solve_parts(A, xy, b, parts)
        assert type(ep.value) is type(e1.value), (name, ep.value, e1.value)
        assert str(ep.value) == str(e1.value), name

"""galerkin_dense (hierarchy.hpp:239-247) on the GPU,
bitwise against the oracle (itself pinned to the reference in
tests/test_oracle.py): random SPD matrices with random surjective partitions
(acceptance.cpp:55-65) and the finest -> level-L partition of a hierarchy."""
import numpy as np
import pytest

import bindings as ob
from paper_1209_5421_b200 import problems

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("trial", range(8))
def test_random_partitions(gpu_api, trial):
    rng = np.random.default_rng(100 + trial)
    n = 16 + 184 * trial // 7
    n_agg = 4 + trial % 13
    A = problems.random_spd(n, 1000 + trial)
    agg = rng.integers(0, n_agg, n).astype(np.int32)
    agg[:n_agg] = np.arange(n_agg)
    assert np.array_equal(gpu_api.galerkin_dense(A, agg, n_agg), ob.galerkin_dense("oracle", A, agg, n_agg))


def test_level_partition_matches_structured_galerkin(gpu_api):
    s = problems.jittered_p1(48)
    h = gpu_api.setup_hierarchy(s.A, s.coords)
    e = h.export()
    agg = e["levels"][0]["agg_of"].astype(np.int32)
    nL = int(e["levels"][1]["n"])
    D = gpu_api.galerkin_dense(s.A, agg, nL)
    assert np.array_equal(D, ob.galerkin_dense("oracle", s.A, agg, nL))
    # the stencil-structured level-L operator holds the same values (hierarchy.hpp:141-192 vs 239-247)
    col, val = e["levels"][1]["ell_col"], e["levels"][1]["ell_val"]
    dense_from_ell = np.zeros((nL, nL))
    for t in range(9):
        for r in range(nL):
            c = col[t * nL + r]
            if c >= 0 and e["levels"][1]["active"][r]:
                dense_from_ell[r, c] = val[t * nL + r]
    act = e["levels"][1]["active"].astype(bool)
    assert np.max(np.abs(D[np.ix_(act, act)] - dense_from_ell[np.ix_(act, act)])) <= 1e-12 * np.max(np.abs(D))


def test_errors(gpu_api):
    A = problems.random_spd(20, 3)
    with pytest.raises(gpu_api.SizeError):
        gpu_api.galerkin_dense(A, np.zeros(19, np.int32), 2)
    with pytest.raises(gpu_api.ArgumentError):
        gpu_api.galerkin_dense(A, np.full(20, 5, np.int32), 2)

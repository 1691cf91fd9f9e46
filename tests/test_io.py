"""File readers: paper_1209_5421_b200 read_matrix_market /
read_mesh / read_coords / write_matrix_market (csrc/io.cpp, multithreaded host
parse) against the reference's own readers (matrix_market.hpp:33-120,
problems.hpp:201-330, built into oracle/_ref): identical arrays bit for bit,
identical exception classes and what() texts (parse_error line numbers), for
the cases of the reference's tests (test_sparse.cpp:263-323,
test_problems.cpp:177-260) plus larger files parsed by many threads."""
import os

import numpy as np
import pytest

import bindings as ob
from paper_1209_5421_b200 import _abi, api

pytestmark = pytest.mark.skipif(not ob.available("ref"), reason="oracle/_ref not built")

STATUS = {1: _abi.SizeError, 4: _abi.ArgumentError, 5: _abi.GeometryError, 8: _abi.IoError, 9: _abi.ParseError}


def _same_csr(a, b):
    assert (a.n_rows, a.n_cols) == (b.n_rows, b.n_cols)
    assert np.array_equal(a.row_ptr, b.row_ptr)
    assert np.array_equal(a.col_idx, b.col_idx)
    assert np.array_equal(a.values.view(np.uint64), b.values.view(np.uint64))


def _write(path, text):
    with open(path, "w") as f:
        f.write(text)
    return str(path)


def _mm_both(path, threads=0):
    st, msg, ref = ob.ref_read_matrix_market(path)
    if st:
        with pytest.raises(STATUS[st]) as ei:
            api.read_matrix_market(path, threads)
        assert str(ei.value) == msg, (str(ei.value), msg)
        return None, (st, msg)
    A = api.read_matrix_market(path, threads)
    _same_csr(A, ref)
    return A, None


@pytest.mark.parametrize("threads", [1, 4, 0])
def test_mm_round_trip_reference_writer(tmp_path, threads):
    """test_sparse.cpp:263-274: read(write(A)) returns A bit for bit."""
    for A in (ob.ref_random_spd(9, 41), ob.ref_make(2, 33, 0.15).A, ob.ref_make(3, 40, 1.3).A):
        p = str(tmp_path / "a.mtx")
        ob.ref_write_matrix_market(A, p)
        B, _ = _mm_both(p, threads)
        _same_csr(B, A)


def test_mm_writer_matches_reference_bytes(tmp_path):
    A = ob.ref_make(3, 24, 1.3).A
    ours, ref = str(tmp_path / "ours.mtx"), str(tmp_path / "ref.mtx")
    api.write_matrix_market(A, ours)
    ob.ref_write_matrix_market(A, ref)
    assert open(ours, "rb").read() == open(ref, "rb").read()


def test_mm_large_file_many_threads(tmp_path):
    """~470K entries: the threaded parse (ranges cut at line starts) gives the
    reference's CSR for every thread count."""
    A = ob.ref_make(2, 257, 0.15).A
    p = str(tmp_path / "big.mtx")
    ob.ref_write_matrix_market(A, p)
    for t in (1, 3, 16):
        B, _ = _mm_both(p, t)
        _same_csr(B, A)


def test_mm_symmetric_storage(tmp_path):
    """test_sparse.cpp:276-295: one triangle stored, both expanded."""
    p = _write(tmp_path / "s.mtx", "%%MatrixMarket matrix coordinate real symmetric\n% lower triangle only\n"
                                   "3 3 4\n1 1 2.0\n2 1 -1.0\n2 2 2.0\n3 3 2.0\n")
    A, _ = _mm_both(p)
    assert A.nnz == 5


MM_CASES = {
    "zero_based": "%%MatrixMarket matrix coordinate real general\n2 2 1\n0 1 3.0\n",
    "array_format": "%%MatrixMarket matrix array real general\n2 2 0\n",
    "bad_banner": "%%MatrixMarkt matrix coordinate real general\n2 2 0\n",
    "complex": "%%MatrixMarket matrix coordinate complex general\n2 2 0\n",
    "hermitian": "%%MatrixMarket matrix coordinate real hermitian\n2 2 0\n",
    "empty": "",
    "no_size": "%%MatrixMarket matrix coordinate real general\n% only comments\n\n",
    "bad_size": "%%MatrixMarket matrix coordinate real general\n2 x 1\n",
    "negative_size": "%%MatrixMarket matrix coordinate real general\n2 2 -1\n",
    "short": "%%MatrixMarket matrix coordinate real general\n3 3 4\n1 1 1.0\n2 2 1.0\n\n% c\n",
    "short_no_newline": "%%MatrixMarket matrix coordinate real general\n3 3 2\n1 1 1.0",
    "malformed": "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n2 x 1.0\n",
    "missing_value": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1\n",
    "inf_value": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 inf\n",
    "overflow": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1e400\n",
    "row_out_of_range": "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n3 1 1.0\n",
    "col_out_of_range": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 3 1.0\n",
    "blank_with_space": "%%MatrixMarket matrix coordinate real general\n2 2 1\n \n1 1 1.0\n",
    "trailing_garbage_after_nnz": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1.0\nnot an entry\n",
    "formats": "%%MatrixMarket MATRIX Coordinate REAL General\n% c\n\n3 3 5\n+1 1 1.5e0\n2 2 -.25\n"
               "3 3 7.\n1 3 1E-3 extra tokens\n3 1 0x1p3\n",
    "duplicates": "%%MatrixMarket matrix coordinate real general\n2 2 4\n1 1 0.1\n2 2 1.0\n1 1 0.2\n1 1 0.3\n",
    "negative_zero": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2 -0.0\n",
    "crlf": "%%MatrixMarket matrix coordinate real general\r\n2 2 2\r\n1 1 1.0\r\n2 2 2.0\r\n",
    "rectangular": "%%MatrixMarket matrix coordinate real general\n2 4 3\n1 4 1.0\n2 1 2.0\n1 1 3.0\n",
}


@pytest.mark.parametrize("name", list(MM_CASES))
def test_mm_cases_match_reference(tmp_path, name):
    _mm_both(_write(tmp_path / f"{name}.mtx", MM_CASES[name]))


def test_mm_parse_error_line(tmp_path):
    """test_sparse.cpp:297-311: the 0-based index is reported at line 3."""
    p = _write(tmp_path / "bad.mtx", MM_CASES["zero_based"])
    with pytest.raises(api.ParseError) as ei:
        api.read_matrix_market(p)
    assert ei.value.line == 3


def test_mm_error_late_in_large_file(tmp_path):
    """The first error in FILE order wins across thread ranges."""
    A = ob.ref_make(2, 129, 0.15).A
    p = str(tmp_path / "a.mtx")
    ob.ref_write_matrix_market(A, p)
    lines = open(p).read().split("\n")
    lines[len(lines) // 3] = "1 1 oops"
    lines[2 * len(lines) // 3] = "0 0 1.0"
    _write(p, "\n".join(lines))
    for t in (1, 8):
        _, err = _mm_both(p, t)
        assert err is not None and err[0] == 9


def test_io_error_missing_file():
    for fn in (api.read_matrix_market, api.read_mesh, api.read_coords):
        with pytest.raises(api.IoError):
            fn("/nonexistent/auxamg.file")
    st, msg, _ = ob.ref_read_matrix_market("/nonexistent/auxamg.mtx")
    with pytest.raises(api.IoError) as ei:
        api.read_matrix_market("/nonexistent/auxamg.mtx")
    assert st == 8 and str(ei.value) == msg


# ------------------------------------------------------------------ meshes
def _mesh_text(mesh, boundary=True):
    out = [f"NODES {len(mesh.nodes)}"]
    out += [f"{i + 1} {x:.17g} {y:.17g}" for i, (x, y) in enumerate(mesh.nodes)]
    out.append(f"ELEMENTS {len(mesh.triangles)}")
    out += [f"{e + 1} {a + 1} {b + 1} {c + 1}" for e, (a, b, c) in enumerate(mesh.triangles)]
    if boundary:
        out.append(f"BOUNDARY {len(mesh.boundary)}")
        ids = [str(i + 1) for i in mesh.boundary]
        out += [" ".join(ids[k:k + 7]) for k in range(0, len(ids), 7)]
    return "\n".join(out) + "\n"


def _mesh_both(path, threads=0):
    st, msg, ref = ob.ref_read_mesh(path)
    if st:
        with pytest.raises(STATUS[st]) as ei:
            api.read_mesh(path, threads)
        assert str(ei.value) == msg, (str(ei.value), msg)
        return None
    m = api.read_mesh(path, threads)
    assert np.array_equal(m.nodes, ref.nodes)
    assert np.array_equal(m.triangles, ref.triangles)
    assert np.array_equal(m.boundary, ref.boundary)
    return m


@pytest.mark.parametrize("kind,n,param", [(1, 2, 0.0), (2, 40, 0.15), (3, 48, 1.3), (4, 40, 0.0)])
@pytest.mark.parametrize("boundary", [True, False])
def test_mesh_round_trip(tmp_path, kind, n, param, boundary):
    """test_problems.cpp:177-196: nodes, triangles and the boundary (explicit
    list or free edges) read back exactly; several thread counts."""
    _, mesh = ob.ref_make(kind, n, param, mesh=True)
    p = _write(tmp_path / "m.mesh", _mesh_text(mesh, boundary))
    for t in (1, 4):
        m = _mesh_both(p, t)
        assert np.array_equal(m.nodes, mesh.nodes) and np.array_equal(m.triangles, mesh.triangles)


MESH_CASES = {
    "vertex_zero": "NODES 3\n1 0 0\n2 1 0\n3 0 1\nELEMENTS 1\n1 0 1 2\n",
    "dup_node": "NODES 3\n1 0 0\n1 1 0\n3 0 1\nELEMENTS 1\n1 1 2 3\n",
    "colinear": "NODES 3\n1 0 0\n2 1 0\n3 2 0\nELEMENTS 1\n1 1 2 3\n",
    "bad_header": "MESH 3\n",
    "no_elements": "NODES 3\n1 0 0\n2 1 0\n3 0 1\n",
    "node_range": "NODES 3\n1 0 0\n4 1 0\n3 0 1\nELEMENTS 1\n1 1 2 3\n",
    "malformed_node": "NODES 3\n1 0 0\n2 1\n3 0 1\nELEMENTS 1\n1 1 2 3\n",
    "dup_then_malformed": "NODES 4\n1 0 0\n1 1 0\n3 0 1\nx\nELEMENTS 1\n1 1 2 3\n",
    "dup_element": "NODES 4\n1 0 0\n2 1 0\n3 0 1\n4 1 1\nELEMENTS 2\n1 1 2 3\n1 2 4 3\n",
    "dup_element_bad_vertex": "NODES 4\n1 0 0\n2 1 0\n3 0 1\n4 1 1\nELEMENTS 2\n1 1 2 3\n1 2 9 3\n",
    "element_range": "NODES 3\n1 0 0\n2 1 0\n3 0 1\nELEMENTS 1\n2 1 2 3\n",
    "blank_lines": "\n  \nNODES 3\n\n1 0 0\n \t\n2 1 0\n3 0 1\n\nELEMENTS 1\n1 1 2 3\n\n",
    "bad_boundary_tag": "NODES 3\n1 0 0\n2 1 0\n3 0 1\nELEMENTS 1\n1 1 2 3\nBND 1\n1\n",
    "boundary_range": "NODES 3\n1 0 0\n2 1 0\n3 0 1\nELEMENTS 1\n1 1 2 3\nBOUNDARY 2\n1 7\n",
    "boundary_short": "NODES 3\n1 0 0\n2 1 0\n3 0 1\nELEMENTS 1\n1 1 2 3\nBOUNDARY 3\n1 2\n",
    "boundary_multi_line": "NODES 4\n1 0 0\n2 1 0\n3 0 1\n4 1 1\nELEMENTS 2\n1 1 2 3\n2 2 4 3\nBOUNDARY 2\n1\n\n4\n",
}


@pytest.mark.parametrize("name", list(MESH_CASES))
def test_mesh_cases_match_reference(tmp_path, name):
    _mesh_both(_write(tmp_path / f"{name}.mesh", MESH_CASES[name]))


def test_mesh_error_line(tmp_path):
    """test_problems.cpp:198-211: vertex id 0 at line 6."""
    p = _write(tmp_path / "bad.mesh", MESH_CASES["vertex_zero"])
    with pytest.raises(api.ParseError) as ei:
        api.read_mesh(p)
    assert ei.value.line == 6


def test_mesh_large_threaded(tmp_path):
    _, mesh = ob.ref_make(2, 200, 0.15, mesh=True)
    p = _write(tmp_path / "big.mesh", _mesh_text(mesh, False))
    for t in (1, 8):
        _mesh_both(p, t)


# ------------------------------------------------------------------ coordinates
COORD_CASES = {
    "basic": "0.5 0.25\n\n1.5 -2.0\n  3 4  \n",
    "oops": "0.5 0.25\noops\n",
    "one_value": "1 2\n3\n",
    "crlf_blank": "1 2\r\n\r\n3 4\r\n",
    "no_trailing_newline": "1 2\n3 4",
    "extra_tokens": "1 2 3\n4 5 junk\n",
}


@pytest.mark.parametrize("name", list(COORD_CASES))
def test_coords_cases_match_reference(tmp_path, name):
    p = _write(tmp_path / f"{name}.xy", COORD_CASES[name])
    st, msg, ref = ob.ref_read_coords(p)
    if st:
        with pytest.raises(STATUS[st]) as ei:
            api.read_coords(p)
        assert str(ei.value) == msg
    else:
        assert np.array_equal(api.read_coords(p), ref)


def test_coords_large_threaded(tmp_path):
    xy = ob.ref_make(2, 300, 0.15).coords
    p = _write(tmp_path / "big.xy", "".join(f"{x:.17g} {y:.17g}\n" for x, y in xy))
    for t in (1, 6):
        assert np.array_equal(api.read_coords(p, t), xy)
    st, _, ref = ob.ref_read_coords(p)
    assert st == 0 and np.array_equal(ref, xy)

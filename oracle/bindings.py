"""oracle/bindings.py — TEST INFRASTRUCTURE ONLY.

ctypes access to the two CPU checkers:
  * "oracle": liboracle.so, the C restatement (oracle/auxamg_oracle.c)
  * "ref":    _ref/libauxamg_ref.so, the unmodified reference headers
              compiled through oracle/ref_shim.cpp

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this.
"""
from __future__ import annotations

import ctypes as C
import os
import sys

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(_HERE))
from paper_1209_5421_b200 import _abi  # noqa: E402

_LIBS = {}


def lib_path(kind: str) -> str:
    """kind: "oracle", "oracle_b256"/"oracle_b64" (dot-blocking sensitivity
    variants of the oracle) or "ref"."""
    if kind.startswith("oracle"):
        return os.path.join(_HERE, "liboracle.so" if kind == "oracle" else f"lib{kind}.so")
    return os.path.join(_HERE, "_ref", "libauxamg_ref.so")


def available(kind: str) -> bool:
    return os.path.exists(lib_path(kind))


def _load(kind: str):
    if kind in _LIBS:
        return _LIBS[kind]
    lib = C.CDLL(lib_path(kind))
    p = "orc_" if kind.startswith("oracle") else "ref_"
    f = lambda name: getattr(lib, p + name)  # noqa: E731
    f("setup").argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.POINTER(C.c_void_p), C.c_char_p, C.c_size_t]
    f("solve").argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_char_p, C.c_size_t]
    f("destroy").argtypes = [C.c_void_p]
    f("n_levels").argtypes = [C.c_void_p]
    for name in ("grid", "stats", "level_info_get", "export_level", "export_coarsest"):
        f(name).restype = C.c_int
    f("grid").argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
    f("stats").argtypes = [C.c_void_p, C.c_void_p]
    f("locality").argtypes = [C.c_void_p, C.c_void_p]
    f("level_info_get").argtypes = [C.c_void_p, C.c_int32, C.c_void_p]
    f("export_level").argtypes = [C.c_void_p, C.c_int32, C.c_void_p]
    f("export_coarsest").argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    f("choose_depth").argtypes = [C.c_long, C.POINTER(C.c_int)]
    f("subregion_of_point").argtypes = [C.c_double, C.c_double, C.c_void_p, C.c_int, C.POINTER(C.c_int)]
    f("point_gs_sweep_ell").argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_char_p, C.c_size_t]
    f("dot").argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
    f("dot").restype = C.c_double
    if kind == "ref":
        lib.ref_set_num_threads.argtypes = [C.c_int]
    _LIBS[kind] = (lib, p)
    return _LIBS[kind]


def csr_view(A):
    v = _abi.CsrView(A.n_rows, A.n_cols, A.nnz, A.row_ptr.ctypes.data, A.col_idx.ctypes.data,
                     A.values.ctypes.data)
    return v


def setup_opts(coarsest_size=64, strict_locality=False, lump_locality=False, symmetry_tol=1e-10):
    return _abi.SetupOpts(coarsest_size, int(strict_locality), int(lump_locality), symmetry_tol)


def cycle_opts(n_inner=2, pre_sweeps=1, post_sweeps=1, max_outer=100, rtol=1e-6, max_directions=0):
    return _abi.CycleOpts(n_inner, pre_sweeps, post_sweeps, max_outer, rtol, max_directions)


class CpuHierarchy:
    """Handle to a hierarchy built by one of the CPU checkers."""

    def __init__(self, kind, A, coords, opts=None):
        self.kind = kind
        self.lib, self.p = _load(kind)
        self._A = A
        coords = np.ascontiguousarray(coords, dtype=np.float64)
        self._xy = coords
        self.h = C.c_void_p()
        msg = C.create_string_buffer(512)
        o = opts if opts is not None else setup_opts()
        s = self._f("setup")(C.byref(csr_view(A)), coords.ctypes.data, coords.shape[0] if coords.ndim == 2 else coords.size // 2,
                             C.byref(o), C.byref(self.h), msg, 512)
        _abi.raise_for(s, msg.raw)

    def _f(self, name):
        return getattr(self.lib, self.p + name)

    def __del__(self):
        try:
            if self.h:
                self._f("destroy")(self.h)
                self.h = C.c_void_p()
        except Exception:
            pass

    def solve(self, b, opts=None, A=None):
        b = np.ascontiguousarray(b, dtype=np.float64)
        o = opts if opts is not None else cycle_opts()
        n = self._A.n_rows
        u = np.zeros(max(n, 1), np.float64)
        hist = np.zeros(o.max_outer + 2, np.float64)
        res = _abi.SolveResultC(u.ctypes.data, hist.ctypes.data, hist.size, 0, 0, 0, 0.0, 0.0, 0.0)
        msg = C.create_string_buffer(512)
        av = C.byref(csr_view(A)) if A is not None else None
        s = self._f("solve")(self.h, av, b.ctypes.data, b.size, C.byref(o), C.byref(res), msg, 512)
        _abi.raise_for(s, msg.raw)
        return {"u": u[:n], "residual_history": hist[: res.history_len].copy(), "iterations": res.iterations,
                "converged": bool(res.converged), "solve_seconds": res.solve_seconds}

    def export(self):
        f = self._f
        return _abi.collect_hierarchy(
            lambda: f("n_levels")(self.h),
            lambda i, o: f("level_info_get")(self.h, i, o),
            lambda i, o: f("export_level")(self.h, i, o),
            lambda box, d: f("grid")(self.h, box, d),
            lambda o: f("locality")(self.h, o),
            lambda o: f("stats")(self.h, o),
            lambda n, lu, perm: f("export_coarsest")(self.h, n, lu, perm),
        )


def set_ref_threads(n: int) -> None:
    lib, _ = _load("ref")
    lib.ref_set_num_threads(n)


def choose_depth(kind, n):
    lib, p = _load(kind)
    d = C.c_int()
    s = getattr(lib, p + "choose_depth")(n, C.byref(d))
    _abi.raise_for(s, b"choose_depth")
    return d.value


def subregion_of_point(kind, x, y, box, k):
    lib, p = _load(kind)
    b = (C.c_double * 4)(*box)
    c = C.c_int()
    s = getattr(lib, p + "subregion_of_point")(x, y, b, k, C.byref(c))
    _abi.raise_for(s, b"subregion_of_point")
    return c.value


def point_gs_sweep_ell(kind, k, col, val, b, x, dir_):
    lib, p = _load(kind)
    x = np.array(x, dtype=np.float64, copy=True)
    msg = C.create_string_buffer(256)
    s = getattr(lib, p + "point_gs_sweep_ell")(k, col.ctypes.data, val.ctypes.data, b.ctypes.data,
                                               x.ctypes.data, dir_, msg, 256)
    _abi.raise_for(s, msg.raw)
    return x


def dot(kind, a, b):
    lib, p = _load(kind)
    return getattr(lib, p + "dot")(a.ctypes.data, b.ctypes.data, a.size)


def galerkin_dense(kind, A, agg_of, n_agg):
    """galerkin_dense (hierarchy.hpp:239-247) through the oracle or the reference."""
    lib, p = _load(kind)
    agg = np.ascontiguousarray(agg_of, dtype=np.int32)
    C_ = np.zeros((n_agg, n_agg), np.float64)
    v = csr_view(A)
    s = getattr(lib, p + "galerkin_dense")(C.byref(v), C.c_void_p(agg.ctypes.data), C.c_int64(agg.size),
                                            C.c_int32(n_agg), C.c_void_p(C_.ctypes.data))
    _abi.raise_for(s, b"galerkin_dense")
    return C_


# ---- the reference's own input generators (problems.hpp, tests/testgen.hpp) via ref_shim.cpp
def _gen_lib():
    lib, _ = _load("ref")
    if not getattr(lib, "_gen_typed", False):
        lib.ref_gen_make.restype = C.c_void_p
        lib.ref_gen_make.argtypes = [C.c_int, C.c_int, C.c_double, C.c_uint, C.c_double]
        lib.ref_gen_random_spd.restype = C.c_void_p
        lib.ref_gen_random_spd.argtypes = [C.c_int, C.c_uint]
        lib.ref_gen_random_stencil.restype = C.c_void_p
        lib.ref_gen_random_stencil.argtypes = [C.c_int, C.c_uint]
        lib.ref_gen_random_vector.argtypes = [C.c_int64, C.c_uint, C.c_double, C.c_double, C.c_void_p]
        for f in ("ref_gen_n", "ref_gen_mesh_nodes", "ref_gen_mesh_tris", "ref_gen_mesh_nboundary"):
            getattr(lib, f).argtypes = [C.c_void_p]
            getattr(lib, f).restype = C.c_int
        for f in ("ref_gen_nnz", "ref_gen_ell_len"):
            getattr(lib, f).argtypes = [C.c_void_p]
            getattr(lib, f).restype = C.c_int64
        for f in ("ref_gen_row_ptr", "ref_gen_col_idx", "ref_gen_ell_col"):
            getattr(lib, f).argtypes = [C.c_void_p]
            getattr(lib, f).restype = C.POINTER(C.c_int32)
        for f in ("ref_gen_values", "ref_gen_b", "ref_gen_xy", "ref_gen_ell_val"):
            getattr(lib, f).argtypes = [C.c_void_p]
            getattr(lib, f).restype = C.POINTER(C.c_double)
        lib.ref_gen_mesh_copy.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        lib.ref_gen_free.argtypes = [C.c_void_p]
        lib._gen_typed = True
    return lib


def _arr(ptr, n, dtype):
    if n == 0:
        return np.zeros(0, dtype)
    return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)


def ref_make(kind: int, n: int, param: float = 0.0, seed: int = 1, jump: float = 0.0, mesh: bool = False):
    """LinearSystem from the reference's own generator (same kinds as
    paper_1209_5421_b200.problems.make); mesh=True also returns the TriMesh."""
    from paper_1209_5421_b200 import problems as P
    lib = _gen_lib()
    h = lib.ref_gen_make(kind, n, param, seed, jump)
    if not h:
        raise ValueError("reference generator failed")
    try:
        N, nnz = lib.ref_gen_n(h), lib.ref_gen_nnz(h)
        A = P.CsrMatrix(N, N, _arr(lib.ref_gen_row_ptr(h), N + 1, np.int32), _arr(lib.ref_gen_col_idx(h), nnz, np.int32),
                        _arr(lib.ref_gen_values(h), nnz, np.float64))
        sysm = P.LinearSystem(A, _arr(lib.ref_gen_b(h), N, np.float64),
                              _arr(lib.ref_gen_xy(h), 2 * N, np.float64).reshape(N, 2))
        if not mesh:
            return sysm
        M, T, B = lib.ref_gen_mesh_nodes(h), lib.ref_gen_mesh_tris(h), lib.ref_gen_mesh_nboundary(h)
        nodes, tris, bnd = np.zeros((M, 2)), np.zeros((T, 3), np.int32), np.zeros(max(B, 1), np.int32)
        lib.ref_gen_mesh_copy(h, nodes.ctypes.data, tris.ctypes.data, bnd.ctypes.data)
        return sysm, P.TriMesh(nodes, tris, bnd[:B])
    finally:
        lib.ref_gen_free(h)


def ref_random_spd(n: int, seed: int):
    from paper_1209_5421_b200 import problems as P
    lib = _gen_lib()
    h = lib.ref_gen_random_spd(n, seed)
    try:
        nnz = lib.ref_gen_nnz(h)
        return P.CsrMatrix(n, n, _arr(lib.ref_gen_row_ptr(h), n + 1, np.int32),
                           _arr(lib.ref_gen_col_idx(h), nnz, np.int32), _arr(lib.ref_gen_values(h), nnz, np.float64))
    finally:
        lib.ref_gen_free(h)


def ref_random_stencil(k: int, seed: int):
    lib = _gen_lib()
    h = lib.ref_gen_random_stencil(k, seed)
    try:
        m = lib.ref_gen_ell_len(h)
        return _arr(lib.ref_gen_ell_col(h), m, np.int32), _arr(lib.ref_gen_ell_val(h), m, np.float64)
    finally:
        lib.ref_gen_free(h)


def ref_random_vector(n: int, seed: int, lo: float = -1.0, hi: float = 1.0):
    out = np.zeros(n, np.float64)
    _gen_lib().ref_gen_random_vector(n, seed, lo, hi, out.ctypes.data)
    return out


# ---- the reference's file readers (matrix_market.hpp, problems.hpp:201-330) via ref_shim.cpp
def _io_lib():
    lib = _gen_lib()
    if not getattr(lib, "_io_typed", False):
        for f in ("ref_read_matrix_market", "ref_read_mesh"):
            getattr(lib, f).argtypes = [C.c_char_p, C.POINTER(C.c_void_p), C.c_char_p, C.c_size_t]
            getattr(lib, f).restype = C.c_int
        lib.ref_read_coords.argtypes = [C.c_char_p, C.POINTER(C.c_void_p), C.POINTER(C.c_int64), C.c_char_p, C.c_size_t]
        lib.ref_read_coords.restype = C.c_int
        lib.ref_write_matrix_market.argtypes = [C.c_void_p, C.c_char_p, C.c_char_p, C.c_size_t]
        lib.ref_write_matrix_market.restype = C.c_int
        lib.ref_gen_ncols.argtypes = [C.c_void_p]
        lib.ref_gen_ncols.restype = C.c_int
        lib._io_typed = True
    return lib


def _ref_status(st, msg):
    """(status, what()) of a reference call; status 0 = no exception."""
    return st, msg.value.decode(errors="replace")


def ref_read_matrix_market(path: str):
    """(status, message, CsrMatrix or None) from auxamg::read_matrix_market."""
    from paper_1209_5421_b200 import problems as P
    lib = _io_lib()
    h, msg = C.c_void_p(), C.create_string_buffer(512)
    st = lib.ref_read_matrix_market(path.encode(), C.byref(h), msg, 512)
    if st:
        return st, msg.value.decode(errors="replace"), None
    try:
        n, m, nnz = lib.ref_gen_n(h), lib.ref_gen_ncols(h), lib.ref_gen_nnz(h)
        A = P.CsrMatrix(n, m, _arr(lib.ref_gen_row_ptr(h), n + 1, np.int32), _arr(lib.ref_gen_col_idx(h), nnz, np.int32),
                        _arr(lib.ref_gen_values(h), nnz, np.float64))
        return 0, "", A
    finally:
        lib.ref_gen_free(h)


def ref_read_mesh(path: str):
    """(status, message, TriMesh or None) from auxamg::read_mesh."""
    from paper_1209_5421_b200 import problems as P
    lib = _io_lib()
    h, msg = C.c_void_p(), C.create_string_buffer(512)
    st = lib.ref_read_mesh(path.encode(), C.byref(h), msg, 512)
    if st:
        return st, msg.value.decode(errors="replace"), None
    try:
        M, T, B = lib.ref_gen_mesh_nodes(h), lib.ref_gen_mesh_tris(h), lib.ref_gen_mesh_nboundary(h)
        nodes, tris, bnd = np.zeros((M, 2)), np.zeros((T, 3), np.int32), np.zeros(max(B, 1), np.int32)
        lib.ref_gen_mesh_copy(h, nodes.ctypes.data, tris.ctypes.data, bnd.ctypes.data)
        return 0, "", P.TriMesh(nodes, tris, bnd[:B])
    finally:
        lib.ref_gen_free(h)


def ref_read_coords(path: str):
    """(status, message, (N, 2) array or None) from auxamg::read_coords."""
    lib = _io_lib()
    h, msg, n = C.c_void_p(), C.create_string_buffer(512), C.c_int64()
    st = lib.ref_read_coords(path.encode(), C.byref(h), C.byref(n), msg, 512)
    if st:
        return st, msg.value.decode(errors="replace"), None
    try:
        return 0, "", _arr(lib.ref_gen_xy(h), 2 * n.value, np.float64).reshape(n.value, 2)
    finally:
        lib.ref_gen_free(h)


def ref_write_matrix_market(A, path: str) -> None:
    lib = _io_lib()
    rp = np.ascontiguousarray(A.row_ptr, np.int32)
    ci = np.ascontiguousarray(A.col_idx, np.int32)
    va = np.ascontiguousarray(A.values, np.float64)

    class _View(C.Structure):
        _fields_ = [("n_rows", C.c_int32), ("n_cols", C.c_int32), ("nnz", C.c_int64),
                    ("row_ptr", C.c_void_p), ("col_idx", C.c_void_p), ("values", C.c_void_p)]
    v = _View(A.n_rows, A.n_cols, int(va.size), rp.ctypes.data, ci.ctypes.data, va.ctypes.data)
    msg = C.create_string_buffer(512)
    st = lib.ref_write_matrix_market(C.byref(v), path.encode(), msg, 512)
    if st:
        raise OSError(msg.value.decode())


def ref_assemble(mesh):
    """LinearSystem from the reference's assemble_fem_triangle (problems.hpp:152-193, f = 1)."""
    from paper_1209_5421_b200 import problems as P
    lib = _io_lib()
    if not getattr(lib, "_asm_typed", False):
        lib.ref_assemble_mesh.restype = C.c_void_p
        lib.ref_assemble_mesh.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_int]
        lib._asm_typed = True
    nd = np.ascontiguousarray(mesh.nodes, np.float64)
    tr = np.ascontiguousarray(mesh.triangles, np.int32)
    bd = np.ascontiguousarray(mesh.boundary, np.int32)
    h = lib.ref_assemble_mesh(nd.ctypes.data, nd.shape[0], tr.ctypes.data, tr.shape[0], bd.ctypes.data, bd.size)
    if not h:
        raise ValueError("reference assembly failed")
    try:
        N, nnz = lib.ref_gen_n(h), lib.ref_gen_nnz(h)
        A = P.CsrMatrix(N, N, _arr(lib.ref_gen_row_ptr(h), N + 1, np.int32), _arr(lib.ref_gen_col_idx(h), nnz, np.int32),
                        _arr(lib.ref_gen_values(h), nnz, np.float64))
        return P.LinearSystem(A, _arr(lib.ref_gen_b(h), N, np.float64),
                              _arr(lib.ref_gen_xy(h), 2 * N, np.float64).reshape(N, 2))
    finally:
        lib.ref_gen_free(h)

"""Synthetic inputs (harness-only): Python view of libauxgen.so
(paper_1209_5421_b200/csrc/problems.cpp), which reproduces the reference's
problem sources (problems.hpp:41-193, tests/testgen.hpp:18-158) and the
BASELINE configurations C1-C5."""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_lib = None

KIND_POISSON5, KIND_SPLIT, KIND_JITTER, KIND_GRADED, KIND_DISK = 0, 1, 2, 3, 4


def _load():
    global _lib
    if _lib is None:
        path = os.path.join(_HERE, "libauxgen.so")
        if not os.path.exists(path):
            raise OSError(f"{path} missing: run __graft_entry__.build()")
        lib = C.CDLL(path)
        lib.auxgen_make.restype = C.c_void_p
        lib.auxgen_make.argtypes = [C.c_int, C.c_int, C.c_double, C.c_uint, C.c_double]
        lib.auxgen_random_spd.restype = C.c_void_p
        lib.auxgen_random_spd.argtypes = [C.c_int, C.c_uint]
        lib.auxgen_random_stencil.restype = C.c_void_p
        lib.auxgen_random_stencil.argtypes = [C.c_int, C.c_uint]
        lib.auxgen_random_vector.argtypes = [C.c_int64, C.c_uint, C.c_double, C.c_double, C.c_void_p]
        for f in ("auxgen_n", "auxgen_mesh_nodes", "auxgen_mesh_tris", "auxgen_mesh_nboundary"):
            getattr(lib, f).argtypes = [C.c_void_p]
            getattr(lib, f).restype = C.c_int
        lib.auxgen_mesh_copy.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        lib.auxgen_nnz.argtypes = [C.c_void_p]
        lib.auxgen_nnz.restype = C.c_int64
        for f in ("auxgen_row_ptr", "auxgen_col_idx", "auxgen_ell_col"):
            getattr(lib, f).argtypes = [C.c_void_p]
            getattr(lib, f).restype = C.POINTER(C.c_int32)
        for f in ("auxgen_values", "auxgen_b", "auxgen_xy", "auxgen_ell_val"):
            getattr(lib, f).argtypes = [C.c_void_p]
            getattr(lib, f).restype = C.POINTER(C.c_double)
        lib.auxgen_free.argtypes = [C.c_void_p]
        _lib = lib
    return _lib


@dataclass
class CsrMatrix:
    """auxamg::CsrMatrix (sparse.hpp:57-74)."""
    n_rows: int
    n_cols: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.values.size)


@dataclass
class LinearSystem:
    """auxamg::LinearSystem (problems.hpp:29-34); coords is (N, 2) float64."""
    A: CsrMatrix
    b: np.ndarray
    coords: np.ndarray


def _copy(ptr, n, dtype):
    if n == 0:
        return np.zeros(0, dtype)
    return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)


def make(kind: int, n: int, param: float = 0.0, seed: int = 1, jump: float = 0.0) -> LinearSystem:
    lib = _load()
    h = lib.auxgen_make(kind, n, param, seed, jump)
    if not h:
        raise ValueError("generator failed")
    try:
        N = lib.auxgen_n(h)
        nnz = lib.auxgen_nnz(h)
        A = CsrMatrix(N, N, _copy(lib.auxgen_row_ptr(h), N + 1, np.int32),
                      _copy(lib.auxgen_col_idx(h), nnz, np.int32),
                      _copy(lib.auxgen_values(h), nnz, np.float64))
        b = _copy(lib.auxgen_b(h), N, np.float64)
        xy = _copy(lib.auxgen_xy(h), 2 * N, np.float64).reshape(N, 2)
    finally:
        lib.auxgen_free(h)
    return LinearSystem(A, b, xy)


def poisson5(n: int) -> LinearSystem:
    """gen_poisson_uniform2d(n) (problems.hpp:41-76)."""
    return make(KIND_POISSON5, n)


def split_p1(n: int, jump: float = 0.0) -> LinearSystem:
    return make(KIND_SPLIT, n, jump=jump)


def jittered_p1(n: int, amp: float = 0.15, seed: int = 1, jump: float = 0.0) -> LinearSystem:
    """Quasi-uniform P1 (BASELINE C1/C3): interior nodes jittered by U(-amp, amp)*h."""
    return make(KIND_JITTER, n, amp, seed, jump)


def graded_p1(n: int, grade: float = 1.3, jump: float = 0.0) -> LinearSystem:
    """testgen::graded_mesh(n, grade) + assemble_fem_triangle (BASELINE C2)."""
    return make(KIND_GRADED, n, grade, jump=jump)


def disk_p1(n: int, radius: float = 0.48) -> LinearSystem:
    """testgen::disk_mesh(n) + assemble_fem_triangle (empty corner cells)."""
    return make(KIND_DISK, n, radius)


def random_spd(n: int, seed: int) -> CsrMatrix:
    lib = _load()
    h = lib.auxgen_random_spd(n, seed)
    try:
        nnz = lib.auxgen_nnz(h)
        return CsrMatrix(n, n, _copy(lib.auxgen_row_ptr(h), n + 1, np.int32),
                         _copy(lib.auxgen_col_idx(h), nnz, np.int32),
                         _copy(lib.auxgen_values(h), nnz, np.float64))
    finally:
        lib.auxgen_free(h)


def random_stencil(k: int, seed: int):
    """testgen::random_stencil(k, seed): (col, val) column-major 9 x 4^k."""
    lib = _load()
    h = lib.auxgen_random_stencil(k, seed)
    try:
        n = 1 << (2 * k)
        return (_copy(lib.auxgen_ell_col(h), 9 * n, np.int32),
                _copy(lib.auxgen_ell_val(h), 9 * n, np.float64))
    finally:
        lib.auxgen_free(h)


def random_vector(n: int, seed: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    lib = _load()
    out = np.zeros(n, np.float64)
    lib.auxgen_random_vector(n, seed, lo, hi, out.ctypes.data)
    return out


@dataclass
class TriMesh:
    """auxamg::TriMesh (problems.hpp:41-47): nodes (M, 2), triangles (T, 3), boundary node ids."""
    nodes: np.ndarray
    triangles: np.ndarray
    boundary: np.ndarray


def make_with_mesh(kind: int, n: int, param: float = 0.0, seed: int = 1, jump: float = 0.0):
    """(LinearSystem, TriMesh) of a P1 kind (1-4): the reference's assembly and its input mesh."""
    lib = _load()
    h = lib.auxgen_make(kind, n, param, seed, jump)
    if not h:
        raise ValueError("generator failed")
    try:
        N = lib.auxgen_n(h)
        nnz = lib.auxgen_nnz(h)
        A = CsrMatrix(N, N, _copy(lib.auxgen_row_ptr(h), N + 1, np.int32),
                      _copy(lib.auxgen_col_idx(h), nnz, np.int32),
                      _copy(lib.auxgen_values(h), nnz, np.float64))
        b = _copy(lib.auxgen_b(h), N, np.float64)
        xy = _copy(lib.auxgen_xy(h), 2 * N, np.float64).reshape(N, 2)
        M, T, B = lib.auxgen_mesh_nodes(h), lib.auxgen_mesh_tris(h), lib.auxgen_mesh_nboundary(h)
        nodes = np.zeros((M, 2))
        tris = np.zeros((T, 3), np.int32)
        bnd = np.zeros(max(B, 1), np.int32)
        lib.auxgen_mesh_copy(h, nodes.ctypes.data, tris.ctypes.data, bnd.ctypes.data)
    finally:
        lib.auxgen_free(h)
    return LinearSystem(A, b, xy), TriMesh(nodes, tris, bnd[:B])

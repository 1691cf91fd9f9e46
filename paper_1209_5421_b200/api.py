"""Python mirror of the reference's C++ solver API, bound to the CUDA library
through the C ABI (include/auxamg_b200.h).

    setup_hierarchy(A, coords, opts)   auxamg::setup_hierarchy   hierarchy.hpp:315-386
    solve(A, b, h, opts)               auxamg::solve             cycle.hpp:202-247
    stats(h)                           auxamg::stats             hierarchy.hpp:395-406
    set_num_threads(n)                 auxamg::set_num_threads   parallel.hpp:43 (no-op)

Same option fields and defaults (SetupOptions hierarchy.hpp:29-34,
CycleOptions cycle.hpp:30-37), same result fields (SolveResult cycle.hpp:47-55)
and the same exception classes (errors.hpp:13-76).  There is no CPU path:
importing this module on a machine without the built library raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from . import _abi
from ._abi import (AuxamgError, SizeError, CapacityError, StructureError, ArgumentError,  # noqa: F401
                   GeometryError, DefinitenessError, SingularError, IoError, ParseError, DeviceError)
from .problems import CsrMatrix, LinearSystem  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))
# AUX_B200_LIB: an alternative build of the same library (A/B timing experiments)
LIB_PATH = os.environ.get("AUX_B200_LIB") or os.path.join(_HERE, "libauxamg_b200.so")
_lib = None


def lib():
    """The loaded CUDA library; raises if it was not built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise OSError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(LIB_PATH)
    vp, i32, i64, sz = C.c_void_p, C.c_int32, C.c_int64, C.c_size_t
    L.aux_setup.argtypes = [vp, vp, i64, vp, vp, C.POINTER(vp), C.c_char_p, sz]
    L.aux_setup_device.argtypes = [vp, vp, i64, vp, vp, C.POINTER(vp), C.c_char_p, sz]
    L.aux_solve.argtypes = [vp, vp, vp, i64, vp, vp, C.c_char_p, sz]
    L.aux_solve_device.argtypes = [vp, vp, i64, vp, vp, C.c_char_p, sz]
    for f in ("aux_setup", "aux_setup_device", "aux_solve", "aux_solve_device", "aux_stats", "aux_get_locality",
              "aux_grid", "aux_level_info_get", "aux_export_level", "aux_export_coarsest", "aux_profile_read",
              "aux_last_timing"):
        getattr(L, f).restype = C.c_int
    L.aux_stats.argtypes = [vp, vp]
    L.aux_get_locality.argtypes = [vp, vp]
    L.aux_grid.argtypes = [vp, vp, vp]
    L.aux_n_levels.argtypes = [vp]
    L.aux_n_levels.restype = i32
    L.aux_level_info_get.argtypes = [vp, i32, vp]
    L.aux_export_level.argtypes = [vp, i32, vp]
    L.aux_export_coarsest.argtypes = [vp, vp, vp, vp]
    L.aux_destroy.argtypes = [vp]
    L.aux_launch_count.restype = i64
    L.aux_profile_enable.argtypes = [vp, i32]
    L.aux_profile_read.argtypes = [vp, i32, C.POINTER(i64), C.POINTER(C.c_double), C.POINTER(C.c_double)]
    L.aux_last_timing.argtypes = [vp, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    L.aux_version.restype = C.c_char_p
    L.aux_set_num_threads.argtypes = [i32]
    L.aux_local_group_create.argtypes = [i32]
    L.aux_local_group_create.restype = vp
    L.aux_local_group_destroy.argtypes = [vp]
    L.aux_nccl_unique_id.argtypes = [vp]
    L.aux_nccl_unique_id.restype = i32
    L.aux_setup_dist.argtypes = [vp, vp, i64, vp, vp, vp, C.POINTER(vp), C.c_char_p, sz]
    L.aux_setup_dist.restype = C.c_int
    L.aux_setup_dist_device.argtypes = [vp, vp, i64, vp, vp, vp, C.POINTER(vp), C.c_char_p, sz]
    L.aux_setup_dist_device.restype = C.c_int
    L.aux_comm_create_nccl.argtypes = [vp, i32, i32, i32]
    L.aux_comm_create_nccl.restype = vp
    L.aux_comm_destroy.argtypes = [vp]
    L.aux_part_dofs.argtypes = [vp, vp]
    L.aux_part_dofs.restype = C.c_int
    L.aux_assemble_p1.argtypes = [vp, i32, vp, i64, vp, i32, C.c_double, C.c_double, i32, C.POINTER(vp),
                                  C.c_char_p, sz]
    L.aux_assemble_p1.restype = C.c_int
    L.aux_system_info.argtypes = [vp, C.POINTER(i32), C.POINTER(i64)]
    L.aux_system_info.restype = C.c_int
    L.aux_system_device.argtypes = [vp, vp, C.POINTER(vp), C.POINTER(vp)]
    L.aux_system_device.restype = C.c_int
    L.aux_system_copy.argtypes = [vp, vp, vp, vp, vp, vp]
    L.aux_system_copy.restype = C.c_int
    L.aux_system_destroy.argtypes = [vp]
    L.aux_galerkin_dense.argtypes = [vp, vp, i64, i32, i32, vp, C.c_char_p, sz]
    L.aux_galerkin_dense.restype = C.c_int
    L.aux_part_rows.argtypes = [vp]
    L.aux_part_rows.restype = i32
    _lib = L
    return L


@dataclass
class SetupOptions:
    """auxamg::SetupOptions (hierarchy.hpp:29-34)."""
    coarsest_size: int = 64
    strict_locality: bool = False
    lump_locality: bool = False
    symmetry_tol: float = 1e-10

    def c(self):
        return _abi.SetupOpts(self.coarsest_size, int(self.strict_locality), int(self.lump_locality),
                              self.symmetry_tol)


@dataclass
class CycleOptions:
    """auxamg::CycleOptions (cycle.hpp:30-37)."""
    n_inner: int = 2
    pre_sweeps: int = 1
    post_sweeps: int = 1
    max_outer: int = 100
    rtol: float = 1e-6
    max_directions: int = 0

    def c(self):
        return _abi.CycleOpts(self.n_inner, self.pre_sweeps, self.post_sweeps, self.max_outer, self.rtol,
                              self.max_directions)


@dataclass
class GpuOptions:
    """B200-only knobs (not part of the reference option structs)."""
    device: int = 0
    coarse_solve: int = 0        # 0 explicit inverse, 1 LU in reference order
    fused_max_cells: int = -1
    use_graphs: bool = True
    block_solve: int = 0         # 0 explicit block inverses, 1 stored LU in reference order
    tile_kernels: bool = True    # overlapped-tile kernels for the structured levels
    cluster_tier: bool = True    # 64x64 level + single-CTA tier in one thread-block cluster
    stream_min_width: int = 0    # row-wavefront kernels from this level width (cells); 0 default, -1 off
    cluster16: bool = True       # 128x128-cell level as one 16-CTA cluster per visit half

    def c(self):
        o = _abi.GpuOpts()
        o.device, o.coarse_solve, o.fused_max_cells, o.use_graphs = (self.device, self.coarse_solve,
                                                                     self.fused_max_cells, int(self.use_graphs))
        o.block_solve = self.block_solve
        o.tile_kernels = int(self.tile_kernels)
        o.cluster_tier = int(self.cluster_tier)
        o.stream_min_width = int(self.stream_min_width)
        o.cluster16 = 0 if self.cluster16 else -1
        return o


@dataclass
class SolveResult:
    """auxamg::SolveResult (cycle.hpp:47-55)."""
    u: np.ndarray
    residual_history: list = field(default_factory=list)
    iterations: int = 0
    converged: bool = False
    setup_seconds: float = 0.0
    solve_seconds: float = 0.0
    total_seconds: float = 0.0


@dataclass
class HierarchyStats:
    """auxamg::HierarchyStats (hierarchy.hpp:388-393)."""
    levels: int
    sizes: list
    nnz: list
    operator_complexity: float


def _csr_view(A: CsrMatrix):
    return _abi.CsrView(A.n_rows, A.n_cols, int(A.values.size), A.row_ptr.ctypes.data,
                        A.col_idx.ctypes.data, A.values.ctypes.data)


def _prep_csr(A: CsrMatrix) -> CsrMatrix:
    return CsrMatrix(int(A.n_rows), int(A.n_cols), np.ascontiguousarray(A.row_ptr, np.int32),
                     np.ascontiguousarray(A.col_idx, np.int32), np.ascontiguousarray(A.values, np.float64))


class Hierarchy:
    """Device-resident auxamg::Hierarchy (hierarchy.hpp:301-309)."""

    def __init__(self, handle, A: CsrMatrix | None, n: int):
        self._h = handle
        self._A = A   # keeps the host arrays alive: solve(A, ...) reuses the device copy
        self.n = n

    @property
    def handle(self):
        return self._h

    def __del__(self):
        try:
            if self._h:
                lib().aux_destroy(self._h)
                self._h = None
        except Exception:
            pass

    def n_levels(self) -> int:
        return lib().aux_n_levels(self._h)

    def stats(self) -> HierarchyStats:
        return stats(self)

    def locality(self):
        loc = _abi.Locality()
        lib().aux_get_locality(self._h, C.byref(loc))
        return loc.dropped, loc.dropped_mass, loc.lumped, loc.lumped_mass

    def export(self) -> dict:
        """Every Hierarchy field in the reference's layout (for parity checks)."""
        L, h = lib(), self._h
        return _abi.collect_hierarchy(
            lambda: L.aux_n_levels(h),
            lambda i, o: L.aux_level_info_get(h, i, o),
            lambda i, o: L.aux_export_level(h, i, o),
            lambda box, d: L.aux_grid(h, box, d),
            lambda o: L.aux_get_locality(h, o),
            lambda o: L.aux_stats(h, o),
            lambda n, lu, perm: L.aux_export_coarsest(h, n, lu, perm),
        )

    def profile(self, on: bool) -> None:
        lib().aux_profile_enable(self._h, int(on))

    def profile_read(self, kind: int):
        n, ms, by = C.c_int64(), C.c_double(), C.c_double()
        _abi.raise_for(lib().aux_profile_read(self._h, kind, C.byref(n), C.byref(ms), C.byref(by)), b"profile")
        return n.value, ms.value, by.value

    def last_timing(self):
        a, b = C.c_double(), C.c_double()
        lib().aux_last_timing(self._h, C.byref(a), C.byref(b))
        return a.value, b.value


def set_num_threads(n: int) -> None:
    lib().aux_set_num_threads(n)


def setup_hierarchy(A: CsrMatrix, coords, opts: SetupOptions | None = None,
                    gpu: GpuOptions | None = None) -> Hierarchy:
    A = _prep_csr(A)
    xy = np.ascontiguousarray(coords, dtype=np.float64)
    npts = xy.shape[0] if xy.ndim == 2 else xy.size // 2
    o = (opts or SetupOptions()).c()
    g = (gpu or GpuOptions()).c()
    h = C.c_void_p()
    msg = C.create_string_buffer(512)
    s = lib().aux_setup(C.byref(_csr_view(A)), xy.ctypes.data, npts, C.byref(o), C.byref(g), C.byref(h), msg, 512)
    _abi.raise_for(s, msg.raw)
    return Hierarchy(h, A, A.n_rows)


def setup_hierarchy_device(n: int, nnz: int, row_ptr: int, col_idx: int, values: int, xy: int, n_points: int,
                           opts: SetupOptions | None = None, gpu: GpuOptions | None = None) -> Hierarchy:
    """setup_hierarchy with every input already in device memory (raw pointers)."""
    v = _abi.CsrView(n, n, nnz, row_ptr, col_idx, values)
    o = (opts or SetupOptions()).c()
    g = (gpu or GpuOptions()).c()
    h = C.c_void_p()
    msg = C.create_string_buffer(512)
    s = lib().aux_setup_device(C.byref(v), xy, n_points, C.byref(o), C.byref(g), C.byref(h), msg, 512)
    _abi.raise_for(s, msg.raw)
    return Hierarchy(h, None, n)


def solve(A: CsrMatrix | None, b, h: Hierarchy, opts: CycleOptions | None = None,
          out: np.ndarray | None = None) -> SolveResult:
    """solve(A, b, h, opts) (cycle.hpp:202-247).  As in the reference, the
    cycle runs on the hierarchy's copy of the setup matrix and the outer A z on
    the caller's A: None or the setup matrix (same arrays and sampled contents,
    or equal contents) reuses the device copy; any other matrix of the same
    order is uploaded for this solve (not on multi-part hierarchies).
    out: optional caller-owned float64 array of length n (e.g. pinned) that
    receives u; the result then references it instead of a fresh copy."""
    o = (opts or CycleOptions()).c()
    b = np.ascontiguousarray(b, dtype=np.float64)
    n = h.n
    if out is not None:
        if out.dtype != np.float64 or not out.flags.c_contiguous or out.size < max(n, 1):
            raise ValueError("out must be a contiguous float64 array of length n")
        u = out
    else:
        u = np.zeros(max(n, 1), np.float64)
    hist = np.zeros(o.max_outer + 2, np.float64)
    res = _abi.SolveResultC(u.ctypes.data, hist.ctypes.data, hist.size, 0, 0, 0, 0.0, 0.0, 0.0)
    msg = C.create_string_buffer(512)
    av = None
    if A is not None:
        if h._A is not None and A is not h._A and _same_arrays(A, h._A):
            A = h._A
        av = C.byref(_csr_view(A if A is h._A else _prep_csr(A)))
    s = lib().aux_solve(h.handle, av, b.ctypes.data, b.size, C.byref(o), C.byref(res), msg, 512)
    _abi.raise_for(s, msg.raw)
    return SolveResult(u[:n] if out is not None else u[:n].copy(), list(hist[: res.history_len]), res.iterations,
                       bool(res.converged), res.setup_seconds, res.solve_seconds, res.total_seconds)


def solve_device(h: Hierarchy, b_ptr: int, u_ptr: int, n: int, opts: CycleOptions | None = None) -> SolveResult:
    """solve() with b and u in device memory (raw pointers, caller DoF order)."""
    o = (opts or CycleOptions()).c()
    hist = np.zeros(o.max_outer + 2, np.float64)
    res = _abi.SolveResultC(u_ptr, hist.ctypes.data, hist.size, 0, 0, 0, 0.0, 0.0, 0.0)
    msg = C.create_string_buffer(512)
    s = lib().aux_solve_device(h.handle, b_ptr, n, C.byref(o), C.byref(res), msg, 512)
    _abi.raise_for(s, msg.raw)
    return SolveResult(None, list(hist[: res.history_len]), res.iterations, bool(res.converged),
                       res.setup_seconds, res.solve_seconds, res.total_seconds)


def _same_arrays(a: CsrMatrix, b: CsrMatrix) -> bool:
    if a.n_rows != b.n_rows or a.values.size != b.values.size:
        return False
    def same_buf(x, y):
        return (x.__array_interface__["data"][0] == y.__array_interface__["data"][0] and x.size == y.size
                and x.dtype == y.dtype)
    if same_buf(a.row_ptr, b.row_ptr) and same_buf(a.col_idx, b.col_idx) and same_buf(a.values, b.values):
        return True   # the setup matrix itself (no O(nnz) host compare)
    return (np.array_equal(a.row_ptr, b.row_ptr) and np.array_equal(a.col_idx, b.col_idx)
            and np.array_equal(a.values, b.values))


def stats(h: Hierarchy) -> HierarchyStats:
    st = _abi.StatsOut()
    lib().aux_stats(h.handle, C.byref(st))
    return HierarchyStats(st.levels, list(st.sizes[: st.levels]), list(st.nnz[: st.levels]),
                          st.operator_complexity)


def launch_count() -> int:
    return lib().aux_launch_count()


# ---------------------------------------------------------------- multi-GPU

class LocalGroup:
    """P parts of one distributed hierarchy driven by P threads of this
    process on one device (the CommLocal transport): the multi-GPU code path,
    runnable on a single B200."""

    def __init__(self, parts: int):
        self.parts = parts
        self._g = lib().aux_local_group_create(parts)
        if not self._g:
            raise _abi.ArgumentError(f"cannot create a local group of {parts} parts")

    def __del__(self):
        try:
            if self._g:
                lib().aux_local_group_destroy(self._g)
                self._g = None
        except Exception:
            pass


class NcclComm:
    """An NCCL communicator (one process per GPU) shared by successive
    distributed hierarchies (transport 2), so setup does not re-initialise NCCL."""

    def __init__(self, nccl_id: bytes, nranks: int, rank: int, device: int = 0):
        buf = (C.c_uint8 * 128).from_buffer_copy(nccl_id)
        self.nranks, self.rank = nranks, rank
        self._c = lib().aux_comm_create_nccl(buf, nranks, rank, device)
        if not self._c:
            raise _abi.DeviceError("NCCL communicator creation failed")

    def __del__(self):
        try:
            if self._c:
                lib().aux_comm_destroy(self._c)
                self._c = None
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    if not lib().aux_nccl_unique_id(buf):
        raise _abi.DeviceError("NCCL unavailable (libnccl.so.2 not found)")
    return bytes(buf)


def setup_hierarchy_dist(A: CsrMatrix, coords, nparts: int, rank: int, group: LocalGroup | None = None,
                         nccl_id: bytes | None = None, opts: SetupOptions | None = None,
                         gpu: GpuOptions | None = None, comm: NcclComm | None = None) -> Hierarchy:
    """setup_hierarchy for part `rank` of `nparts` (A and coords are the global
    inputs).  group: local transport (threads, one device); nccl_id: NCCL, one
    process per GPU."""
    A = _prep_csr(A)
    xy = np.ascontiguousarray(coords, dtype=np.float64)
    npts = xy.shape[0] if xy.ndim == 2 else xy.size // 2
    d = _abi.DistOpts()
    d.nparts, d.rank = nparts, rank
    if comm is not None:
        d.transport, d.local_group = 2, comm._c
    elif group is not None:
        d.transport, d.local_group = 0, group._g
    else:
        if nccl_id is None or len(nccl_id) != 128:
            raise _abi.ArgumentError("setup_hierarchy_dist: need a LocalGroup or a 128-byte NCCL id")
        d.transport = 1
        C.memmove(d.nccl_id, nccl_id, 128)
    o = (opts or SetupOptions()).c()
    g = (gpu or GpuOptions()).c()
    h = C.c_void_p()
    msg = C.create_string_buffer(512)
    s = lib().aux_setup_dist(C.byref(_csr_view(A)), xy.ctypes.data, npts, C.byref(o), C.byref(g), C.byref(d),
                             C.byref(h), msg, 512)
    _abi.raise_for(s, msg.raw)
    hh = Hierarchy(h, A, A.n_rows)
    hh._transport = comm if comm is not None else group   # outlives the hierarchy
    return hh


def setup_hierarchy_dist_device(n: int, nnz: int, row_ptr: int, col_idx: int, values: int, xy: int, n_points: int,
                                nparts: int, rank: int, group: LocalGroup | None = None,
                                nccl_id: bytes | None = None, opts: SetupOptions | None = None,
                                gpu: GpuOptions | None = None, comm: NcclComm | None = None) -> Hierarchy:
    """setup_hierarchy_dist with the global inputs already in device memory."""
    v = _abi.CsrView(n, n, nnz, row_ptr, col_idx, values)
    d = _abi.DistOpts()
    d.nparts, d.rank = nparts, rank
    if comm is not None:
        d.transport, d.local_group = 2, comm._c
    elif group is not None:
        d.transport, d.local_group = 0, group._g
    else:
        if nccl_id is None or len(nccl_id) != 128:
            raise _abi.ArgumentError("setup_hierarchy_dist_device: need a LocalGroup or a 128-byte NCCL id")
        d.transport = 1
        C.memmove(d.nccl_id, nccl_id, 128)
    o = (opts or SetupOptions()).c()
    g = (gpu or GpuOptions()).c()
    h = C.c_void_p()
    msg = C.create_string_buffer(512)
    s = lib().aux_setup_dist_device(C.byref(v), xy, n_points, C.byref(o), C.byref(g), C.byref(d), C.byref(h), msg,
                                    512)
    _abi.raise_for(s, msg.raw)
    hh = Hierarchy(h, None, n)
    hh._transport = comm if comm is not None else group
    return hh


def part_rows(h: Hierarchy) -> int:
    return lib().aux_part_rows(h.handle)


def part_dofs(h: Hierarchy) -> np.ndarray:
    """Caller ids of the finest DoFs this part owns."""
    ids = np.empty(max(part_rows(h), 1), np.int32)
    _abi.raise_for(lib().aux_part_dofs(h.handle, ids.ctypes.data), b"aux_part_dofs")
    return ids[: part_rows(h)]


def solve_parts(A: CsrMatrix, coords, b, parts: int, opts: SetupOptions | None = None,
                cycle: CycleOptions | None = None, gpu: GpuOptions | None = None):
    """Set up and solve with `parts` parts on this process's device (local
    transport, one thread per part).  Returns (u assembled from the parts'
    owned entries, list of per-part SolveResult, list of per-part stats)."""
    import threading
    grp = LocalGroup(parts)
    u = np.zeros(A.n_rows)
    results, stats_, errors = [None] * parts, [None] * parts, [None] * parts

    def run(r):
        try:
            h = setup_hierarchy_dist(A, coords, parts, r, group=grp, opts=opts, gpu=gpu)
            stats_[r] = h.stats()
            results[r] = solve(A, b, h, cycle, out=u)
            del h
        except Exception as e:   # noqa: BLE001 - re-raised below
            errors[r] = e

    th = [threading.Thread(target=run, args=(r,)) for r in range(parts)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for e in errors:
        if e is not None:
            raise e
    return u, results, stats_


# ---------------------------------------------------------------- device assembly

class DeviceSystem:
    """A P1 system assembled on the GPU (aux_assemble_p1), resident in device memory."""

    def __init__(self, nodes, triangles, boundary, f: float = 1.0, jump: float = 0.0, device: int = 0):
        nd = np.ascontiguousarray(nodes, dtype=np.float64)
        tr = np.ascontiguousarray(triangles, dtype=np.int32)
        bd = np.ascontiguousarray(boundary, dtype=np.int32)
        h = C.c_void_p()
        msg = C.create_string_buffer(512)
        s = lib().aux_assemble_p1(nd.ctypes.data, nd.shape[0], tr.ctypes.data, tr.shape[0], bd.ctypes.data,
                                  bd.size, f, jump, device, C.byref(h), msg, 512)
        _abi.raise_for(s, msg.raw)
        self._s = h
        n, nnz = C.c_int32(), C.c_int64()
        lib().aux_system_info(h, C.byref(n), C.byref(nnz))
        self.n, self.nnz = n.value, nnz.value

    def device_view(self):
        """(aux_csr_view with device pointers, b pointer, coordinates pointer)."""
        v = _abi.CsrView()
        b, xy = C.c_void_p(), C.c_void_p()
        lib().aux_system_device(self._s, C.byref(v), C.byref(b), C.byref(xy))
        return v, b.value, xy.value

    def to_host(self):
        """(CsrMatrix, b, coords) copied to the host."""
        rp = np.empty(self.n + 1, np.int32)
        col = np.empty(max(self.nnz, 1), np.int32)
        val = np.empty(max(self.nnz, 1), np.float64)
        b = np.empty(max(self.n, 1), np.float64)
        xy = np.empty((max(self.n, 1), 2), np.float64)
        _abi.raise_for(lib().aux_system_copy(self._s, rp.ctypes.data, col.ctypes.data, val.ctypes.data,
                                             b.ctypes.data, xy.ctypes.data), b"aux_system_copy")
        return CsrMatrix(self.n, self.n, rp, col[: self.nnz], val[: self.nnz]), b[: self.n], xy[: self.n]

    def setup(self, opts: SetupOptions | None = None, gpu: GpuOptions | None = None) -> Hierarchy:
        """setup_hierarchy straight from the device-resident system."""
        v, _, xy = self.device_view()
        o = (opts or SetupOptions()).c()
        g = (gpu or GpuOptions()).c()
        h = C.c_void_p()
        msg = C.create_string_buffer(512)
        s = lib().aux_setup_device(C.byref(v), xy, self.n, C.byref(o), C.byref(g), C.byref(h), msg, 512)
        _abi.raise_for(s, msg.raw)
        hh = Hierarchy(h, None, self.n)
        hh._system = self   # the device arrays outlive nothing they are needed for, but keep them
        return hh

    def __del__(self):
        try:
            if self._s:
                lib().aux_system_destroy(self._s)
                self._s = None
        except Exception:
            pass


def galerkin_dense(A: CsrMatrix, agg_of, n_agg: int, device: int = 0) -> np.ndarray:
    """galerkin_dense (hierarchy.hpp:239-247) on the GPU: dense P^T A P for an arbitrary partition."""
    A = _prep_csr(A)
    agg = np.ascontiguousarray(agg_of, dtype=np.int32)
    out = np.zeros((n_agg, n_agg), np.float64)
    msg = C.create_string_buffer(512)
    s = lib().aux_galerkin_dense(C.byref(_csr_view(A)), agg.ctypes.data, agg.size, n_agg, device, out.ctypes.data,
                                 msg, 512)
    _abi.raise_for(s, msg.raw)
    return out


# ---------------------------------------------------------------- file readers
def _file_lib():
    L = lib()
    if not getattr(L, "_io_typed", False):
        vp, sz = C.c_void_p, C.c_size_t
        for f in ("aux_read_matrix_market", "aux_read_mesh", "aux_read_coords"):
            getattr(L, f).argtypes = [C.c_char_p, C.c_int32, C.POINTER(vp), C.c_char_p, sz]
            getattr(L, f).restype = C.c_int
        L.aux_file_data_sizes.argtypes = [vp, vp, vp, vp]
        L.aux_file_data_sizes.restype = C.c_int
        L.aux_file_data_copy.argtypes = [vp, vp, vp, vp]
        L.aux_file_data_copy.restype = C.c_int
        L.aux_file_data_destroy.argtypes = [vp]
        L.aux_write_matrix_market.argtypes = [vp, C.c_char_p, C.c_char_p, sz]
        L.aux_write_matrix_market.restype = C.c_int
        L._io_typed = True
    return L


def _read(fn: str, path: str, threads: int):
    L = _file_lib()
    h, msg = C.c_void_p(), C.create_string_buffer(512)
    st = getattr(L, fn)(os.fsencode(path), threads, C.byref(h), msg, 512)
    _abi.raise_for(st, msg.raw)
    a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
    L.aux_file_data_sizes(h, C.byref(a), C.byref(b), C.byref(c))
    return L, h, a.value, b.value, c.value


def read_matrix_market(path: str, threads: int = 0) -> CsrMatrix:
    """read_matrix_market (matrix_market.hpp:33-104): coordinate real general /
    symmetric, 1-based; symmetric storage expanded; parsed by `threads` host
    threads (0: all)."""
    L, h, n, m, nnz = _read("aux_read_matrix_market", path, threads)
    try:
        rp, ci, va = np.empty(n + 1, np.int32), np.empty(nnz, np.int32), np.empty(nnz, np.float64)
        L.aux_file_data_copy(h, rp.ctypes.data, ci.ctypes.data, va.ctypes.data)
        return CsrMatrix(int(n), int(m), rp, ci, va)
    finally:
        L.aux_file_data_destroy(h)


def read_mesh(path: str, threads: int = 0):
    """read_mesh (problems.hpp:201-310): NODES / ELEMENTS / optional BOUNDARY;
    the boundary is the explicit list united with the free edges' endpoints."""
    from .problems import TriMesh
    L, h, nn, ne, nb = _read("aux_read_mesh", path, threads)
    try:
        nodes, tris, bnd = np.empty((nn, 2)), np.empty((ne, 3), np.int32), np.empty(nb, np.int32)
        L.aux_file_data_copy(h, nodes.ctypes.data, tris.ctypes.data, bnd.ctypes.data)
        return TriMesh(nodes, tris, bnd)
    finally:
        L.aux_file_data_destroy(h)


def read_coords(path: str, threads: int = 0) -> np.ndarray:
    """read_coords (problems.hpp:313-330): one "x y" per non-blank line, (N, 2)."""
    L, h, n, _, _ = _read("aux_read_coords", path, threads)
    try:
        xy = np.empty((n, 2))
        L.aux_file_data_copy(h, xy.ctypes.data, None, None)
        return xy
    finally:
        L.aux_file_data_destroy(h)


def write_matrix_market(A: CsrMatrix, path: str) -> None:
    """write_matrix_market (matrix_market.hpp:106-120): general, %.17g values."""
    A = _prep_csr(A)
    msg = C.create_string_buffer(512)
    st = _file_lib().aux_write_matrix_market(C.byref(_csr_view(A)), os.fsencode(path), msg, 512)
    _abi.raise_for(st, msg.raw)

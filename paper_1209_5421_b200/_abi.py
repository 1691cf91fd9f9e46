"""ctypes mirror of include/auxamg_b200.h (structs, status codes, exceptions).

The exception classes mirror the reference hierarchy in errors.hpp:13-76
(`auxamg::error` and its subclasses) so Python callers see the same error
types the C++ API throws.
"""
from __future__ import annotations

import ctypes as C

AUX_MAX_LEVELS = 40


class AuxamgError(RuntimeError):
    """auxamg::error (errors.hpp:13-16)."""


class SizeError(AuxamgError):
    """auxamg::size_error (errors.hpp:19-22)."""


class CapacityError(AuxamgError):
    """auxamg::capacity_error (errors.hpp:25-28)."""


class StructureError(AuxamgError):
    """auxamg::structure_error (errors.hpp:31-34)."""


class ArgumentError(AuxamgError):
    """auxamg::argument_error (errors.hpp:37-40)."""


class GeometryError(AuxamgError):
    """auxamg::geometry_error (errors.hpp:43-46)."""


class DefinitenessError(AuxamgError):
    """auxamg::definiteness_error (errors.hpp:49-52)."""


class SingularError(AuxamgError):
    """auxamg::singular_error (errors.hpp:55-58)."""


class IoError(AuxamgError):
    """auxamg::io_error (errors.hpp:61-64)."""


class ParseError(AuxamgError):
    """auxamg::parse_error (errors.hpp:67-76); .line is the 1-based line number."""

    @property
    def line(self) -> int:
        import re
        m = re.search(r"\(line (-?\d+)\)$", str(self))
        return int(m.group(1)) if m else -1


class DeviceError(AuxamgError):
    """CUDA failure inside the B200 library (no reference analogue)."""


STATUS_TO_EXC = {
    1: SizeError,
    2: CapacityError,
    3: StructureError,
    4: ArgumentError,
    5: GeometryError,
    6: DefinitenessError,
    7: SingularError,
    8: IoError,
    9: ParseError,
    100: DeviceError,
    101: AuxamgError,
}


def raise_for(status: int, msg: bytes | str = b"") -> None:
    if status == 0:
        return
    if isinstance(msg, (bytes, bytearray)):
        msg = msg.split(b"\0", 1)[0].decode(errors="replace")
    raise STATUS_TO_EXC.get(status, AuxamgError)(msg)


class CsrView(C.Structure):
    _fields_ = [("n_rows", C.c_int32), ("n_cols", C.c_int32), ("nnz", C.c_int64),
                ("row_ptr", C.c_void_p), ("col_idx", C.c_void_p), ("values", C.c_void_p)]


class SetupOpts(C.Structure):
    _fields_ = [("coarsest_size", C.c_int32), ("strict_locality", C.c_int32),
                ("lump_locality", C.c_int32), ("symmetry_tol", C.c_double)]


class CycleOpts(C.Structure):
    _fields_ = [("n_inner", C.c_int32), ("pre_sweeps", C.c_int32), ("post_sweeps", C.c_int32),
                ("max_outer", C.c_int32), ("rtol", C.c_double), ("max_directions", C.c_int32)]


class GpuOpts(C.Structure):
    _fields_ = [("device", C.c_int32), ("coarse_solve", C.c_int32), ("fused_max_cells", C.c_int32),
                ("use_graphs", C.c_int32), ("block_solve", C.c_int32),
                ("tile_kernels", C.c_int32), ("cluster_tier", C.c_int32), ("stream_min_width", C.c_int32),
                ("cluster16", C.c_int32)]


class DistOpts(C.Structure):
    """aux_dist_opts: one part of a multi-GPU hierarchy."""
    _fields_ = [("nparts", C.c_int32), ("rank", C.c_int32), ("transport", C.c_int32), ("reserved", C.c_int32),
                ("local_group", C.c_void_p), ("nccl_id", C.c_uint8 * 128)]


class Locality(C.Structure):
    _fields_ = [("dropped", C.c_int64), ("dropped_mass", C.c_double),
                ("lumped", C.c_int64), ("lumped_mass", C.c_double)]


class StatsOut(C.Structure):
    _fields_ = [("levels", C.c_int32), ("sizes", C.c_int64 * AUX_MAX_LEVELS),
                ("nnz", C.c_int64 * AUX_MAX_LEVELS), ("operator_complexity", C.c_double)]


class SolveResultC(C.Structure):
    _fields_ = [("u", C.c_void_p), ("residual_history", C.c_void_p), ("history_capacity", C.c_int32),
                ("history_len", C.c_int32), ("iterations", C.c_int32), ("converged", C.c_int32),
                ("setup_seconds", C.c_double), ("solve_seconds", C.c_double),
                ("total_seconds", C.c_double)]


class LevelInfo(C.Structure):
    _fields_ = [("k", C.c_int32), ("structured", C.c_int32), ("n", C.c_int32), ("nnz", C.c_int64),
                ("has_map", C.c_int32), ("map_level", C.c_int32), ("n_aggregates", C.c_int32),
                ("n_items", C.c_int32), ("block_pool", C.c_int64)]


class LevelExport(C.Structure):
    _fields_ = [("agg_of", C.c_void_p), ("member_ptr", C.c_void_p), ("member_idx", C.c_void_p),
                ("active", C.c_void_p), ("item_color", C.c_void_p), ("ell_col", C.c_void_p),
                ("ell_val", C.c_void_p), ("block_size", C.c_void_p), ("block_offset", C.c_void_p),
                ("block_lu", C.c_void_p), ("block_perm", C.c_void_p)]


def ptr(a) -> C.c_void_p:
    """Raw data pointer of a C-contiguous numpy array (or None)."""
    if a is None:
        return None
    return C.c_void_p(a.ctypes.data)


def collect_hierarchy(n_levels, level_info, export_level, grid, locality, stats, coarsest):
    """Export every field of a Hierarchy (hierarchy.hpp:288-309) into numpy
    arrays, in the reference's indexing and layout.  The callables take the
    same arguments as the aux_* C functions minus the handle."""
    import numpy as np

    out = {"levels": []}
    box = (C.c_double * 4)()
    depth = C.c_int32()
    grid(box, C.byref(depth))
    out["box"] = tuple(box)
    out["depth"] = depth.value
    loc = Locality()
    locality(C.byref(loc))
    out["locality"] = (loc.dropped, loc.dropped_mass, loc.lumped, loc.lumped_mass)
    st = StatsOut()
    stats(C.byref(st))
    out["stats"] = {"levels": st.levels, "sizes": list(st.sizes[: st.levels]),
                    "nnz": list(st.nnz[: st.levels]), "operator_complexity": st.operator_complexity}
    for i in range(n_levels()):
        info = LevelInfo()
        s = level_info(i, C.byref(info))
        raise_for(s, b"level_info")
        n, na, ni = info.n, info.n_aggregates, info.n_items
        lv = {"k": info.k, "structured": bool(info.structured), "n": n, "nnz": info.nnz,
              "has_map": bool(info.has_map)}
        ex = LevelExport()
        arrs = {}
        if info.has_map:
            arrs["map_level"] = info.map_level
            arrs["n_aggregates"] = na
            arrs["agg_of"] = np.zeros(n, np.int32)
            arrs["member_ptr"] = np.zeros(na + 1, np.int32)
            arrs["member_idx"] = np.zeros(n, np.int32)
        arrs["active"] = np.zeros(n, np.uint8)
        arrs["item_color"] = np.zeros(ni, np.int32)
        if info.structured:
            arrs["ell_col"] = np.zeros(9 * n, np.int32)
            arrs["ell_val"] = np.zeros(9 * n, np.float64)
        if not info.structured and info.has_map:
            arrs["block_size"] = np.zeros(na, np.int32)
            arrs["block_offset"] = np.zeros(na + 1, np.int64)
            arrs["block_lu"] = np.zeros(max(info.block_pool, 1), np.float64)
            arrs["block_perm"] = np.zeros(max(n, 1), np.int32)
        for name, _ in LevelExport._fields_:
            if name in arrs:
                setattr(ex, name, arrs[name].ctypes.data)
        raise_for(export_level(i, C.byref(ex)), b"export_level")
        lv.update(arrs)
        out["levels"].append(lv)
    nc = C.c_int32()
    coarsest(C.byref(nc), None, None)
    lu = np.zeros(nc.value * nc.value, np.float64)
    perm = np.zeros(nc.value, np.int32)
    coarsest(C.byref(nc), lu.ctypes.data, perm.ctypes.data)
    out["coarsest_lu"] = lu.reshape(nc.value, nc.value)
    out["coarsest_perm"] = perm
    return out

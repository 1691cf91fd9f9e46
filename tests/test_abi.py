"""CPU tests of the boundary: the C-ABI library loads (no GPU needed) and
exports every symbol include/auxamg_b200.h declares; the Python mirror keeps
the reference's option defaults and exception classes."""
import ctypes
import os
import re

import pytest

from paper_1209_5421_b200 import _abi, api

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "auxamg_b200.h")).read()
    return sorted(set(re.findall(r"\b(aux_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(api.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_defaults_match_reference():
    lib = api.lib()
    so = _abi.SetupOpts()
    lib.aux_default_setup_opts(ctypes.byref(so))
    assert (so.coarsest_size, so.strict_locality, so.lump_locality, so.symmetry_tol) == (64, 0, 0, 1e-10)
    co = _abi.CycleOpts()
    lib.aux_default_cycle_opts(ctypes.byref(co))
    assert (co.n_inner, co.pre_sweeps, co.post_sweeps, co.max_outer, co.rtol, co.max_directions) == (2, 1, 1, 100, 1e-6, 0)
    d = api.SetupOptions()
    assert (d.coarsest_size, d.strict_locality, d.lump_locality, d.symmetry_tol) == (64, False, False, 1e-10)
    c = api.CycleOptions()
    assert (c.n_inner, c.pre_sweeps, c.post_sweeps, c.max_outer, c.rtol, c.max_directions) == (2, 1, 1, 100, 1e-6, 0)


def test_status_codes_map_to_reference_exceptions():
    assert issubclass(api.SizeError, api.AuxamgError)
    for code, exc in _abi.STATUS_TO_EXC.items():
        with pytest.raises(exc):
            _abi.raise_for(code, b"x")
    _abi.raise_for(0, b"")


def test_version_string():
    assert b"sm_100a" in api.lib().aux_version()


def test_no_gpu_setup_fails_loudly():
    """Without a device the product path raises (no CPU fallback)."""
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except Exception:
        pass
    from paper_1209_5421_b200 import problems
    s = problems.poisson5(10)
    with pytest.raises(api.AuxamgError):
        api.setup_hierarchy(s.A, s.coords)


def test_dist_transport_validated_before_any_device_work():
    """aux_dist_opts.transport outside {0, 1, 2} is an argument_error (no
    device work: this runs without a GPU)."""
    import ctypes as C
    import numpy as np
    from paper_1209_5421_b200 import _abi, api
    rp = np.array([0, 1], np.int32)
    ci = np.array([0], np.int32)
    va = np.array([1.0])
    xy = np.zeros(2)
    v = _abi.CsrView(1, 1, 1, rp.ctypes.data, ci.ctypes.data, va.ctypes.data)
    d = _abi.DistOpts()
    d.nparts, d.rank, d.transport = 1, 0, 7
    h = C.c_void_p()
    msg = C.create_string_buffer(256)
    st = api.lib().aux_setup_dist(C.byref(v), xy.ctypes.data, 1, None, None, C.byref(d), C.byref(h), msg, 256)
    assert _abi.STATUS_TO_EXC[st] is _abi.ArgumentError, (st, msg.value)
    assert b"transport" in msg.value

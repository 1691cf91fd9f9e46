"""The ctypes mirrors of the C ABI structs (paper_1209_5421_b200/_abi.py) have
the layout of include/auxamg_b200.h: a small C program compiled with gcc
prints sizeof / offsetof of every field, compared with the ctypes fields.
(A drifted field would pass options or read results at the wrong offsets.)"""
import os
import shutil
import subprocess
import tempfile

import pytest

from paper_1209_5421_b200 import _abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

STRUCTS = {
    "aux_csr_view": _abi.CsrView,
    "aux_setup_opts": _abi.SetupOpts,
    "aux_cycle_opts": _abi.CycleOpts,
    "aux_gpu_opts": _abi.GpuOpts,
    "aux_dist_opts": _abi.DistOpts,
    "aux_locality": _abi.Locality,
    "aux_stats_out": _abi.StatsOut,
    "aux_solve_result": _abi.SolveResultC,
    "aux_level_info": _abi.LevelInfo,
    "aux_level_export": _abi.LevelExport,
}


@pytest.fixture(scope="module")
def c_layout():
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "auxamg_b200.h"', "int main(void) {"]
    for cname, cls in STRUCTS.items():
        lines.append(f'  printf("{cname} size %zu\\n", sizeof({cname}));')
        for f in cls._fields_:
            lines.append(f'  printf("{cname} {f[0]} %zu\\n", offsetof({cname}, {f[0]}));')
    lines += ["  return 0;", "}"]
    d = tempfile.mkdtemp()
    src, exe = os.path.join(d, "layout.c"), os.path.join(d, "layout")
    open(src, "w").write("\n".join(lines) + "\n")
    subprocess.run(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), src, "-o", exe], check=True)
    out = subprocess.run([exe], check=True, capture_output=True, text=True).stdout
    shutil.rmtree(d, ignore_errors=True)
    res = {}
    for ln in out.splitlines():
        name, field, val = ln.split()
        res[(name, field)] = int(val)
    return res


@pytest.mark.parametrize("cname", list(STRUCTS))
def test_struct_layout_matches_header(c_layout, cname):
    cls = STRUCTS[cname]
    assert c_layout[(cname, "size")] == _abi.C.sizeof(cls), cname
    for f in cls._fields_:
        assert c_layout[(cname, f[0])] == getattr(cls, f[0]).offset, (cname, f[0])

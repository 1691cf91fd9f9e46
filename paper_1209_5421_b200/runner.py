"""Batch runner with a backend switch.

Mirrors the reference's runner (runner.hpp:87-197) and CLI (auxamg_cli.cpp:26-50)
for generator sources: build the problem, run setup + solve, emit the same CSV
(`N,levels,opcomplexity,iters,setup_s,solve_s,total_s,converged`), residual CSV
(`N,iter,residual`) and JSON-lines reports, with `--backend b200` (this
library; `--gpus P` runs the multi-GPU path, P parts on this process's device)
or `--backend reference` (the reference compiled in place, oracle/_ref).

    python -m paper_1209_5421_b200.runner --gen poisson2d --n 257 --n 513 --format csv
    python -m paper_1209_5421_b200.runner --gen graded --n 2049 --backend b200 --format jsonl

Sources as in load_problem (runner.hpp:64-83): `--gen` (the reference's
`poisson2d` plus the harness families of SURVEY 8(d): `split`, `jitter`,
`graded`, `disk`, `jump`), `--matrix F --coords F` (Matrix Market + one "x y"
line per DoF, b = 1) or `--mesh F` (P1 assembly, f = 1) -- files parsed by the
library's multithreaded readers (csrc/io.cpp); with the b200 backend a mesh
is assembled on the GPU (aux_assemble_p1).  `--gpus P` runs the multi-GPU
code path with P parts of one process on this process's device (the
in-process transport); one process per GPU is bench.py's torchrun path.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
from dataclasses import dataclass, field

import numpy as np

from . import problems

GENERATORS = {
    "poisson2d": lambda n: problems.poisson5(n),      # gen_poisson_uniform2d (runner.hpp:57-61)
    "split": lambda n: problems.split_p1(n),
    "jitter": lambda n: problems.jittered_p1(n),
    "graded": lambda n: problems.graded_p1(n, 1.3),
    "disk": lambda n: problems.disk_p1(n),
    "jump": lambda n: problems.jittered_p1(n, jump=1e3),
}


@dataclass
class RunReport:
    """auxamg::RunReport (runner.hpp:41-53)."""
    label: str
    n: int = 0
    nnz: int = 0
    levels: int = 0
    level_sizes: list = field(default_factory=list)
    level_nnz: list = field(default_factory=list)
    opcomplexity: float = 0.0
    iters: int = 0
    converged: bool = False
    setup_s: float = 0.0
    solve_s: float = 0.0
    total_s: float = 0.0
    residual_history: list = field(default_factory=list)


def _solve_b200(sysm, gpus, setup_opts, cycle_opts):
    from . import api
    if gpus <= 1:
        t1 = time.perf_counter()
        h = api.setup_hierarchy(sysm.A, sysm.coords, setup_opts)
        setup_s = time.perf_counter() - t1
        st = h.stats()
        r = api.solve(sysm.A, sysm.b, h, cycle_opts)
        return st, r, setup_s
    t1 = time.perf_counter()
    u, res, stats = api.solve_parts(sysm.A, sysm.coords, sysm.b, gpus, setup_opts, cycle_opts)
    wall = time.perf_counter() - t1
    r = res[0]
    r.u = u
    return stats[0], r, wall - r.solve_seconds


def _solve_reference(sysm, setup_opts, cycle_opts, threads):
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
    import bindings as ob
    from . import api
    ob.set_ref_threads(threads)
    so = ob.setup_opts(setup_opts.coarsest_size, setup_opts.strict_locality, setup_opts.lump_locality,
                       setup_opts.symmetry_tol)
    co = ob.cycle_opts(cycle_opts.n_inner, cycle_opts.pre_sweeps, cycle_opts.post_sweeps, cycle_opts.max_outer,
                       cycle_opts.rtol, cycle_opts.max_directions)
    t1 = time.perf_counter()
    h = ob.CpuHierarchy("ref", sysm.A, sysm.coords, so)
    setup_s = time.perf_counter() - t1
    e = h.export()
    st = api.HierarchyStats(e["stats"]["levels"], list(e["stats"]["sizes"]), list(e["stats"]["nnz"]),
                            e["stats"]["operator_complexity"])
    r = h.solve(sysm.b, co)
    res = api.SolveResult(r["u"], list(r["residual_history"]), r["iterations"], bool(r["converged"]), setup_s,
                          r.get("solve_seconds", 0.0), 0.0)
    return st, res, setup_s


def load_problem(gen: str | None, size: int, matrix: str = "", coords: str = "", mesh: str = "",
                 backend: str = "b200", threads: int = 0) -> problems.LinearSystem:
    """load_problem (runner.hpp:64-83): one source -> LinearSystem."""
    from . import api
    if gen:
        if gen not in GENERATORS:
            raise api.ArgumentError(f"unknown generator '{gen}'")
        return GENERATORS[gen](size)
    if matrix:
        if not coords:
            raise api.ArgumentError("--matrix requires --coords (the method needs DoF coordinates)")
        A = api.read_matrix_market(matrix, threads)
        xy = api.read_coords(coords, threads)
        if xy.shape[0] != A.n_rows:
            raise api.SizeError("coordinate count does not match matrix order")
        return problems.LinearSystem(A, np.ones(A.n_rows), xy)
    m = api.read_mesh(mesh, threads)
    if backend == "b200":   # assemble_fem_triangle on the GPU
        A, b, xy = api.DeviceSystem(m.nodes, m.triangles, m.boundary).to_host()
        return problems.LinearSystem(A, b, xy)
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
    import bindings as ob
    return ob.ref_assemble(m)


def run_one(gen: str | None, size: int, backend: str = "b200", gpus: int = 1, setup_opts=None, cycle_opts=None,
            threads: int = 1, matrix: str = "", coords: str = "", mesh: str = "") -> RunReport:
    """run_one (runner.hpp:87-112): problem, setup, stats, solve, timings."""
    from . import api
    setup_opts = setup_opts or api.SetupOptions()
    cycle_opts = cycle_opts or api.CycleOptions()
    t0 = time.perf_counter()
    sysm = load_problem(gen, size, matrix, coords, mesh, backend)
    label = f"{gen}-{size}" if gen else (matrix or mesh)
    rep = RunReport(label=label, n=sysm.A.n_rows, nnz=sysm.A.nnz)
    if backend == "b200":
        st, r, setup_s = _solve_b200(sysm, gpus, setup_opts, cycle_opts)
    elif backend == "reference":
        st, r, setup_s = _solve_reference(sysm, setup_opts, cycle_opts, threads)
    else:
        raise api.ArgumentError(f"unknown backend '{backend}'")
    rep.setup_s = setup_s
    rep.levels = st.levels
    rep.level_sizes = list(st.sizes)[: st.levels]
    rep.level_nnz = list(st.nnz)[: st.levels]
    rep.opcomplexity = st.operator_complexity
    rep.solve_s = r.solve_seconds
    rep.iters = r.iterations
    rep.converged = r.converged
    rep.residual_history = list(r.residual_history)
    rep.total_s = time.perf_counter() - t0
    return rep


def write_csv(reports, out) -> None:
    """write_csv (runner.hpp:131-141): the same header and number formats."""
    out.write("N,levels,opcomplexity,iters,setup_s,solve_s,total_s,converged\n")
    for r in reports:
        out.write(f"{r.n},{r.levels},{r.opcomplexity:.4f},{r.iters},{r.setup_s:.3f},{r.solve_s:.3f},"
                  f"{r.total_s:.3f},{1 if r.converged else 0}\n")


def write_residuals(reports, out) -> None:
    """write_residuals (runner.hpp:144-153)."""
    out.write("N,iter,residual\n")
    for r in reports:
        for i, v in enumerate(r.residual_history):
            out.write(f"{r.n},{i},{v:.17g}\n")


def write_jsonl(reports, out) -> None:
    """write_jsonl (runner.hpp:155-173): one JSON object per run, the same keys."""
    for r in reports:
        out.write(json.dumps({"label": r.label, "n": r.n, "nnz": r.nnz, "levels": r.levels,
                              "level_sizes": r.level_sizes, "level_nnz": r.level_nnz,
                              "opcomplexity": r.opcomplexity, "iters": r.iters, "converged": r.converged,
                              "setup_s": r.setup_s, "solve_s": r.solve_s, "total_s": r.total_s,
                              "residual_history": r.residual_history}) + "\n")


def main(argv=None) -> int:
    from . import api
    ap = argparse.ArgumentParser(description="auxamg batch runner with a B200 backend")
    ap.add_argument("--gen", default="")
    ap.add_argument("--n", type=int, action="append", default=[])
    ap.add_argument("--matrix", default="")
    ap.add_argument("--coords", default="")
    ap.add_argument("--mesh", default="")
    ap.add_argument("--backend", default="b200", choices=["b200", "reference"])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--threads", type=int, default=1)
    ap.add_argument("--format", default="csv", choices=["csv", "jsonl"])
    ap.add_argument("--report", default="")
    ap.add_argument("--residuals", default="")
    ap.add_argument("--rtol", type=float, default=1e-6)
    ap.add_argument("--max-outer", type=int, default=100)
    ap.add_argument("--n-inner", type=int, default=2)
    ap.add_argument("--coarsest", type=int, default=64)
    a = ap.parse_args(argv)
    try:
        co = api.CycleOptions(n_inner=a.n_inner, max_outer=a.max_outer, rtol=a.rtol)
        so = api.SetupOptions(coarsest_size=a.coarsest)
        if sum(bool(x) for x in (a.gen, a.matrix, a.mesh)) != 1:
            raise api.ArgumentError("exactly one of --gen, --matrix, --mesh must be given")
        if a.gen and not a.n:
            raise api.ArgumentError("--gen requires at least one --n")
        if a.gen:
            reports = [run_one(a.gen, n, a.backend, a.gpus, so, co, a.threads) for n in a.n]
        else:
            reports = [run_one(None, 0, a.backend, a.gpus, so, co, a.threads, a.matrix, a.coords, a.mesh)]
    except api.ArgumentError as e:   # auxamg_cli.cpp:83-92: argument errors -> 1, others -> 3
        print(f"error: {e}", file=sys.stderr)
        return 1
    except api.AuxamgError as e:
        print(f"error: {e}", file=sys.stderr)
        return 3
    out = open(a.report, "w") if a.report else sys.stdout
    (write_csv if a.format == "csv" else write_jsonl)(reports, out)
    if a.report:
        out.close()
    if a.format == "csv" and (a.residuals or a.report):
        path = a.residuals or os.path.splitext(a.report)[0] + "_residuals.csv"
        with open(path, "w") as f:
            write_residuals(reports, f)
    return 0


if __name__ == "__main__":
    raise SystemExit(main())

"""bench.py — setup+solve ms/MDOF of the B200 auxiliary-grid AMG.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--config c1|c2|c3|c4|c5] [--no-cpu-baseline]

Default workload at N=1: BASELINE config C3, the largest single-GPU
configuration (2D P1 Poisson on the quasi-uniform jittered split mesh, n=4097,
N = 16,777,216, rtol 1e-6).  For N > 1 (torchrun) the default is the C5
weak-scaling family (5-point Poisson, n = 4097, 5794, 8193, 11586 for
1/2/4/8 GPUs, ~16.8M DoFs per GPU), solved as ONE coupled problem: quadtree-
subtree partition, NCCL ghost / ring exchange and all-reduced inner products,
coarse levels agglomerated on rank 0.

One "step" = setup_hierarchy + solve of the whole problem (the north-star path,
hierarchy.hpp:315-386 + cycle.hpp:202-247).  `value` is measured with the
inputs (CSR, coordinates, b) already resident in HBM, through the device entry
points of the C ABI; `e2e` is the same step through the host-buffer C ABI
(aux_setup / aux_solve) with the host->device copies of A, coords and b from
pinned memory and the device->host copy of u inside the timed region.
`--impl reference` times the reference's own CPU implementation (oracle/_ref,
the unmodified reference headers compiled in place, fed by the reference's own
generators) on the host cores, on the same `config`.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "setup+solve ms/MDOF, 2D P1 Poisson to 1e-6 rel res; SpMV/smoother HBM GB/s"

# kind numbers of problems.make / bindings.ref_make
CONFIGS = {
    "c1": dict(kind=2, n=1025, param=0.15, jump=0.0,
               name="C1: P1 Poisson on quasi-uniform (jittered) split mesh n=1025, N=1,048,576"),
    "c2": dict(kind=3, n=2049, param=1.3, jump=0.0,
               name="C2: P1 Poisson on graded_mesh(2049,1.3) (shape-regular, locally refined), N=4,194,304"),
    "c3": dict(kind=2, n=4097, param=0.15, jump=0.0,
               name="C3: P1 Poisson on quasi-uniform (jittered) split mesh n=4097, N=16,777,216"),
    "c4": dict(kind=2, n=4097, param=0.15, jump=1e3,
               name="C4: P1 jump-coefficient diffusion (kappa 1/1e3, 8x8 checkerboard) on the C3 mesh, N=16,777,216"),
    "c5": dict(kind=0, n=4097, param=0.0, jump=0.0,
               name="C5: 5-point Poisson n=4097, N=16,777,216 (weak-scaling family, 1 GPU point)"),
}
# C5 weak scaling: global n per GPU count, ~16.8M DoFs per GPU
WEAK_N = {1: 4097, 2: 5794, 4: 8193, 8: 11586}
REF_BUDGET_S = 150.0   # reference arm: whole run bounded to a few minutes
PROFILE_KINDS = {0: "finest block Gauss-Seidel colour pass (k_bgs_inv)",
                 1: "finest CSR SpMV + fused dots (k_csr_spmv)",
                 2: "finest residual + restriction (k_rows + k_restrict_cells)",
                 3: "coarse K-cycle below the finest level (graph replay per finest visit)",
                 4: "level-L 9-point pre-smoothing GS + residual + restriction (k_stream_down; k_tile_down below 1024 cells wide)",
                 5: "level-L 9-point post-smoothing GS + ELL SpMV + dots (k_stream_up; k_tile_up below 1024 cells wide)"}


def scaled(cfg, world):
    """The workload at `world` GPUs (weak scaling: DoFs per GPU fixed)."""
    if world == 1:
        return cfg
    cfg = dict(cfg)
    cfg["n"] = WEAK_N.get(world, int(round((cfg["n"] - 1) * world ** 0.5)) + 1) if cfg["kind"] == 0 \
        else int(round((cfg["n"] - 1) * world ** 0.5)) + 1
    N = (cfg["n"] - 1) ** 2
    cfg["name"] = (f"C5: 5-point Poisson weak scaling, n={cfg['n']}, N={N:,} on {world} GPUs"
                   if cfg["kind"] == 0 else f"{cfg['name']} x{world} GPUs weak scaling (global n={cfg['n']})")
    return cfg


def make_problem(cfg):
    from paper_1209_5421_b200 import problems
    return problems.make(cfg["kind"], cfg["n"], cfg["param"], 1, cfg["jump"])


L2_BYTES = 126e6


def input_bytes(N, nnz):
    return 12 * nnz + 4 * (N + 1) + 24 * N


def needs_flush(N, nnz):
    """Inputs that fit the 126 MB L2 twice over get an explicit L2 flush before every timed step."""
    return input_bytes(N, nnz) < 2 * L2_BYTES


def config_dict(cfg, N, nnz):
    """The `config` object, identical in both arms."""
    inputs = input_bytes(N, nnz)
    l2 = (f"inputs {inputs / 1e6:.0f} MB > 2 x 126 MB L2 (no flush needed)" if not needs_flush(N, nnz) else
          f"inputs {inputs / 1e6:.0f} MB < 2 x 126 MB L2: a 256 MB buffer is written (L2 flush) before every timed step")
    return {"workload": cfg["name"], "N": int(N), "nnz": int(nnz), "rtol": 1e-6, "l2": l2}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        q = ("index,clocks.sm,clocks.max.sm," + os.environ.get("AUX_SMI_POWER", "power.draw") + ",clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            if os.environ.get("AUX_SMI_OFF"):
                raise RuntimeError("sampler off")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", os.environ.get("AUX_SMI_MS", "500")],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        # let nvidia-smi finish starting up (NVML init, first sample) before the
        # timed region opens: its start-up competes with the driver calls of the
        # first timed steps (seen as a 5-8 ms per-step gap on some boxes)
        t_end = time.time() + 3.0
        while self.proc is not None and time.time() < t_end:
            try:
                if os.path.getsize(self.path) > 0:
                    break
            except OSError:
                break
            time.sleep(0.02)
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            for line in open(self.path):
                f = [x.strip() for x in line.split(",")]
                if len(f) < 9:
                    continue
                try:
                    sm.append(float(f[1]))
                    mx.append(float(f[2]))
                except ValueError:
                    continue
                for nm, v in zip(names, f[5:9]):
                    if v.lower().startswith("active"):
                        reasons.add(nm)
            os.unlink(self.path)
        except Exception:
            pass
        load = [s for s in sm if mx and s > 0.5 * max(mx)] or sm
        return {"sm_mhz": statistics.median(load) if load else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist  # noqa: F811
        import torch
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    return world, rank, local, dist


def _ref_solve_once(ob, s, threads):
    ob.set_ref_threads(threads)
    t0 = time.perf_counter()
    h = ob.CpuHierarchy("ref", s.A, s.coords)
    r = h.solve(s.b)
    dt = time.perf_counter() - t0
    del h
    return dt, r["iterations"]


def run_reference(args, cfg, world, rank):
    """--impl reference: the reference's own CPU path on the host cores, fed by
    the reference's own generators (no repo library is mapped).  Each step is
    one full setup_hierarchy + solve; the number of timed steps is bounded so
    the whole run ends within a few minutes (REF_BUDGET_S)."""
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import bindings as ob
    if not ob.available("ref"):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libauxamg_ref.so not built"}))
        return
    threads = os.cpu_count() or 1
    s = ob.ref_make(cfg["kind"], cfg["n"], cfg["param"], 1, cfg["jump"])
    N, nnz = s.A.n_rows, s.A.nnz
    mdof = N / 1e6
    t_start = time.perf_counter()
    dt, iters = _ref_solve_once(ob, s, threads)   # first run: warm-up, and sizes the sample
    warm = 1
    budget = max(REF_BUDGET_S - (time.perf_counter() - t_start), dt)
    steps = max(1, min(args.steps, int(budget // max(dt, 1e-9))))
    extra_warm = min(max(args.warmup - 1, 0), max(0, int(budget // max(dt, 1e-9)) - steps))
    for _ in range(extra_warm):
        _ref_solve_once(ob, s, threads)
        warm += 1
    times = []
    for _ in range(steps):
        t, iters = _ref_solve_once(ob, s, threads)
        times.append(t)
    ms = 1e3 * statistics.median(times)
    val = ms / mdof
    out = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "ms/MDOF", "n_gpus": world,
        "steps": len(times), "warmup": warm, "ms_per_step": ms, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (the reference's own generators)",
        "config": config_dict(cfg, N, nnz), "iterations": iters,
        "parallelism": f"host CPU, {threads} threads (auxamg::set_num_threads)",
        "cpu_baseline": {"value": val, "unit": "ms/MDOF", "cores": threads, "kind": "reference",
                         "sample": (f"full workload setup_hierarchy+solve, median of {len(times)} "
                                    f"(steps bounded to ~{REF_BUDGET_S:.0f} s of CPU time; requested {args.steps})")},
        "e2e": {"value": val, "unit": "ms/MDOF", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out))


def cpu_baseline(s, threads):
    """The reference itself (oracle/_ref; the C port when it is absent) on the
    same inputs: one full setup_hierarchy + solve with `threads` threads."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import bindings as ob
    kind = "ref" if ob.available("ref") else "oracle"
    if kind == "ref":
        ob.set_ref_threads(threads)
    else:
        threads = 1   # the C restatement is single-threaded
    t0 = time.perf_counter()
    h = ob.CpuHierarchy(kind, s.A, s.coords)
    r = h.solve(s.b)
    dt = time.perf_counter() - t0
    del h
    return {"value": 1e3 * dt / (s.A.n_rows / 1e6), "unit": "ms/MDOF", "cores": threads,
            "kind": "reference" if kind == "ref" else "port",
            "sample": f"one full setup_hierarchy+solve of the same workload ({r['iterations']} iterations)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS),
                    help="default: c3 on one GPU, the c5 weak-scaling family on several")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-weak-base", action="store_true",
                    help="skip the 1-GPU C5 point reported next to the N=1 line")
    ap.add_argument("--dist", action="store_true",
                    help="use the multi-GPU (NCCL) path even on one GPU (it is always used for --gpus > 1)")
    args = ap.parse_args()
    world, rank, local, dist = dist_setup(args)
    cfg_name = args.config or ("c3" if world == 1 else "c5")
    cfg = scaled(CONFIGS[cfg_name], world)
    if args.impl == "reference":
        run_reference(args, cfg, world, rank)
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return

    import torch
    from paper_1209_5421_b200 import api

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    api.lib()
    use_dist = world > 1 or args.dist
    gpu = api.GpuOptions(device=local)
    comm = None
    if use_dist:   # one NCCL communicator for every hierarchy of the run
        nid = api.nccl_unique_id() if rank == 0 else bytes(128)
        if dist is not None:
            obj = [nid]
            dist.broadcast_object_list(obj, src=0)
            nid = obj[0]
        comm = api.NcclComm(nid, world, rank, local)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def maxr(v):
        if dist is None:
            return v
        t = torch.tensor([v], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def measure(s, steps, warmup, with_profile):
        """Device-resident and end-to-end setup+solve of one system."""
        N, nnz = s.A.n_rows, s.A.nnz
        d_rp = torch.from_numpy(s.A.row_ptr).to(dev)
        d_col = torch.from_numpy(s.A.col_idx).to(dev)
        d_val = torch.from_numpy(s.A.values).to(dev)
        d_xy = torch.from_numpy(np.ascontiguousarray(s.coords)).to(dev)
        d_b = torch.from_numpy(s.b).to(dev)
        d_u = torch.empty(N, dtype=torch.float64, device=dev)

        def setup_dev():
            if use_dist:
                return api.setup_hierarchy_dist_device(N, nnz, d_rp.data_ptr(), d_col.data_ptr(), d_val.data_ptr(),
                                                       d_xy.data_ptr(), N, world, rank, comm=comm, gpu=gpu)
            return api.setup_hierarchy_device(N, nnz, d_rp.data_ptr(), d_col.data_ptr(), d_val.data_ptr(),
                                              d_xy.data_ptr(), N, gpu=gpu)

        def setup_host(A_h, xy_h):
            if use_dist:
                return api.setup_hierarchy_dist(A_h, xy_h, world, rank, comm=comm, gpu=gpu)
            return api.setup_hierarchy(A_h, xy_h, gpu=gpu)

        for _ in range(warmup):
            h = setup_dev()
            api.solve_device(h, d_b.data_ptr(), d_u.data_ptr(), N)
            del h
        barrier()
        launches0 = api.launch_count()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        iters = None
        setup_ms, solve_ms = [], []
        step_ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if needs_flush(N, nnz) else None

        def l2_flush(k):
            if flush is not None:   # (the library's own stream starts after this completes)
                flush.fill_(k & 0xff)
                torch.cuda.current_stream().synchronize()

        l2_flush(0)   # the fill kernel loads lazily: not inside the timed region
        with ClockSampler(local) as clk:
            barrier()
            ev0.record()
            for k in range(steps):
                l2_flush(k)
                step_ev[k].record()
                h = setup_dev()
                r = api.solve_device(h, d_b.data_ptr(), d_u.data_ptr(), N)
                iters = r.iterations
                a, b = h.last_timing()
                setup_ms.append(a)
                solve_ms.append(b)
                del h
            step_ev[steps].record()
            ev1.record()
            barrier()
        launches = api.launch_count() - launches0
        ms_step = maxr(ev0.elapsed_time(ev1)) / steps
        steps_ms = [round(step_ev[k].elapsed_time(step_ev[k + 1]), 3) for k in range(steps)]
        u_dev = d_u.cpu().numpy()
        prof = {}
        if with_profile:
            # untimed solves with CUDA events around the profiled kernels on their
            # launch stream: mode 1 (graph replay of the coarse cycle) for the
            # finest kernels and the coarse share, mode 2 (eager) for level L
            h = setup_dev()
            h.profile(1)
            api.solve_device(h, d_b.data_ptr(), d_u.data_ptr(), N)
            for kind in (0, 1, 2, 3):
                prof[kind] = h.profile_read(kind)
            h.profile(2)
            api.solve_device(h, d_b.data_ptr(), d_u.data_ptr(), N)
            for kind in (4, 5):
                prof[kind] = h.profile_read(kind)
            h.profile(0)
            del h
        # e2e through the host-buffer C ABI, pinned memory
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
        A_h = api.CsrMatrix(N, N, pin(s.A.row_ptr), pin(s.A.col_idx), pin(s.A.values))
        xy_h, b_h = pin(s.coords), pin(s.b)
        u_h = pin(np.zeros(N))
        h2d = A_h.row_ptr.nbytes + A_h.col_idx.nbytes + A_h.values.nbytes + xy_h.nbytes + b_h.nbytes
        for _ in range(max(1, warmup // 2)):
            h = setup_host(A_h, xy_h)
            api.solve(A_h, b_h, h, out=u_h)
            del h
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for k in range(steps):
            l2_flush(k)
            h = setup_host(A_h, xy_h)
            res = api.solve(A_h, b_h, h, out=u_h)
            del h
        e1.record()
        barrier()
        e2e_ms = maxr(e0.elapsed_time(e1)) / steps
        if use_dist:   # each part wrote the entries of the DoFs it owns
            hq = setup_dev()
            ids = api.part_dofs(hq)
            del hq
            assert np.array_equal(res.u[ids], u_dev[ids]), "host-API and device-API solutions differ"
        else:
            assert np.array_equal(res.u, u_dev), "host-API and device-API solutions differ"
        return dict(ms_step=ms_step, e2e_ms=e2e_ms, iters=iters, launches=launches, clocks=clk.summary(), steps_ms=steps_ms,
                    setup_ms=statistics.median(setup_ms), solve_ms=statistics.median(solve_ms), prof=prof,
                    h2d=int(h2d), d2h=int(N * 8))

    s = make_problem(cfg)
    N, nnz = s.A.n_rows, s.A.nnz
    mdof = N / 1e6
    m = measure(s, args.steps, args.warmup, True)
    value = m["ms_step"] / mdof   # whole-job: the global problem (all GPUs' DoFs) per step

    # ---- rooflines from the live CUDA events (algorithmic bytes, SURVEY 8(d) / DESIGN.md §4)
    peak, peak_src = peaks()
    prof = m["prof"]
    solve_ms = m["solve_ms"]
    kernels = {}
    for k, (n_l, tot_ms, bytes_l) in prof.items():
        ent = {"launches": n_l, "ms_total": round(tot_ms, 4),
               "us_per_launch": round(1e3 * tot_ms / n_l, 3) if n_l else None}
        if k != 3 and n_l:
            ach = bytes_l / (tot_ms / n_l * 1e-3) / 1e9
            ent.update({"algorithmic_bytes_per_launch": bytes_l, "achieved_gbs": round(ach, 1),
                        "frac": round(ach / peak, 4)})
        if k <= 3:
            ent["share_of_solve"] = round(tot_ms / solve_ms, 4)
        else:
            ent["note"] = "eager launches (profile mode 2); in the timed graph replay they run back to back"
        kernels[PROFILE_KINDS[k]] = ent
    kind = max((0, 1, 2), key=lambda k: prof[k][1])   # dominant HBM-bound kernel of the timed solve
    n_l, tot_ms, bytes_l = prof[kind]
    achieved = bytes_l / (tot_ms / n_l * 1e-3) / 1e9 if n_l else 0.0
    traffic, tdb = None, {}
    try:   # ncu DRAM read+write bytes per launch (tools/traffic_from_ncu.py)
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tdb = json.load(f).get(cfg_name, {})
        traffic = tdb.get(str(kind))
    except Exception:
        pass
    for k, ent in zip(prof, kernels.values()):
        if str(k) in tdb:
            ent["traffic"] = tdb[str(k)]

    out = {
        "metric": METRIC, "value": value, "unit": "ms/MDOF", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": m["ms_step"], "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (generators pinned byte-identical to the reference's)",
        "config": config_dict(cfg, N, nnz), "iterations": m["iters"],
        "parallelism": (f"quadtree-subtree partition over {world} GPUs, NCCL halo/ghost exchange + all-reduce, "
                        "coarse levels agglomerated on rank 0") if use_dist else "1 GPU",
        "breakdown": {"setup_ms": m["setup_ms"], "solve_ms": solve_ms, "steps_ms": m["steps_ms"],
                      "coarse_kcycle_ms": round(prof[3][1], 3) if 3 in prof else None},
        "e2e": {"value": m["e2e_ms"] / mdof, "unit": "ms/MDOF", "h2d_bytes_per_step": m["h2d"],
                "d2h_bytes_per_step": m["d2h"]},
        "roofline": {"bound": "hbm", "kernel": PROFILE_KINDS[kind], "achieved": achieved, "peak": peak,
                     "peak_source": peak_src, "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                     "launches": n_l, "algorithmic_bytes_per_launch": bytes_l, "kernels": kernels},
        "gpu_launches": int(m["launches"]),
        "clocks": m["clocks"],
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(s, os.cpu_count() or 1)
        out["cpu_baseline_1thread"] = cpu_baseline(s, 1)
    if world == 1 and not args.no_weak_base and cfg_name != "c5":
        # the 1-GPU point of the C5 weak-scaling family (the --gpus N runs use it)
        del s
        s5 = make_problem(CONFIGS["c5"])
        m5 = measure(s5, max(2, args.steps // 2), min(args.warmup, 3), False)
        out["weak_scaling_base"] = {"workload": CONFIGS["c5"]["name"], "value": m5["ms_step"] / (s5.A.n_rows / 1e6),
                                    "e2e": m5["e2e_ms"] / (s5.A.n_rows / 1e6), "iterations": m5["iters"],
                                    "unit": "ms/MDOF"}
        del s5
    if rank == 0:
        print(json.dumps(out))
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

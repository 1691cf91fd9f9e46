"""bench.py — setup+solve ms/MDOF of the B200 auxiliary-grid AMG on BASELINE
config C2 (2D P1 Poisson on graded_mesh(2049, 1.3), N = 4,194,304, rtol 1e-6).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--config c2|c1|c3]

One "step" = setup_hierarchy + solve of the whole problem (the north-star path,
hierarchy.hpp:315-386 + cycle.hpp:202-247).  `value` is measured with the
inputs (CSR, coordinates, b) already resident in HBM, through the device entry
points of the C ABI; `e2e` is the same step through the host-buffer C ABI
(aux_setup / aux_solve) with the host->device copies of A, coords and b from
pinned memory and the device->host copy of u inside the timed region.
Multi-GPU (torchrun): every rank solves its own replica of the workload
(weak scaling; coupled domain decomposition is not implemented yet).
`--impl reference` times the reference's own CPU implementation (oracle/_ref,
the unmodified reference headers compiled in place) on the host cores.
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

CONFIGS = {
    "c2": dict(kind="graded", n=2049, param=1.3,
               name="C2: P1 Poisson on graded_mesh(2049,1.3) (shape-regular, locally refined), N=4,194,304"),
    "c1": dict(kind="jitter", n=1025, param=0.15,
               name="C1: P1 Poisson on quasi-uniform (jittered) split mesh n=1025, N=1,048,576"),
    "c3": dict(kind="jitter", n=4097, param=0.15,
               name="C3: P1 Poisson on quasi-uniform (jittered) split mesh n=4097, N=16,777,216"),
}
PROFILE_KINDS = {0: "finest block Gauss-Seidel colour pass (k_bgs*)", 1: "finest CSR SpMV + fused dots (k_csr_spmv)",
                 2: "finest residual + restriction (k_csr_resid_restrict)"}


def make_problem(cfg):
    from paper_1209_5421_b200 import problems
    if cfg["kind"] == "graded":
        return problems.graded_p1(cfg["n"], cfg["param"])
    return problems.jittered_p1(cfg["n"], cfg["param"])


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
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
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


def run_reference(args, cfg, world, rank):
    """--impl reference: the reference's own CPU path on the host cores."""
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import bindings as ob
    if not ob.available("ref"):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libauxamg_ref.so not built"}))
        return
    threads = os.cpu_count() or 1
    ob.set_ref_threads(threads)
    s = make_problem(cfg)
    mdof = s.A.n_rows / 1e6
    times, iters = [], None
    warm, steps = args.warmup, args.steps
    it = 0
    while it < warm + steps:
        t0 = time.perf_counter()
        h = ob.CpuHierarchy("ref", s.A, s.coords)
        r = h.solve(s.b)
        dt = time.perf_counter() - t0
        del h
        iters = r["iterations"]
        if it >= warm:
            times.append(dt)
        if it == 0 and dt > 40.0:   # keep the whole run within a few minutes: this run is the sample
            times.append(dt)
            warm, steps = 0, 1
            break
        it += 1
    ms = 1e3 * statistics.median(times)
    val = ms / mdof
    out = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "ms/MDOF", "n_gpus": world,
        "steps": len(times), "warmup": warm, "ms_per_step": ms, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["name"], "iterations": iters, "rtol": 1e-6},
        "cpu_baseline": {"value": val, "unit": "ms/MDOF", "cores": threads, "kind": "reference",
                         "sample": f"full workload ({cfg['name']}) setup_hierarchy+solve, median of {len(times)}"},
        "e2e": {"value": val, "unit": "ms/MDOF", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out))


def cpu_baseline(cfg, s):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import bindings as ob
    kind = "ref" if ob.available("ref") else "oracle"
    threads = os.cpu_count() or 1 if kind == "ref" else 1
    if kind == "ref":
        ob.set_ref_threads(threads)
    t0 = time.perf_counter()
    h = ob.CpuHierarchy(kind, s.A, s.coords)
    r = h.solve(s.b)
    dt = time.perf_counter() - t0
    return {"value": 1e3 * dt / (s.A.n_rows / 1e6), "unit": "ms/MDOF", "cores": threads,
            "kind": "reference" if kind == "ref" else "port",
            "sample": f"one full setup_hierarchy+solve of the same workload ({r['iterations']} iterations)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dist", action="store_true",
                    help="use the multi-GPU (NCCL) path even on one GPU (it is always used for --gpus > 1)")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    world, rank, local, dist = dist_setup(args)
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
    if world > 1:   # weak scaling: the global problem grows with the GPU count (same DoFs per GPU)
        cfg = dict(cfg)
        cfg["n"] = int(round((cfg["n"] - 1) * world ** 0.5)) + 1
        cfg["name"] = f"{cfg['name']} x{world} GPUs weak scaling (global n={cfg['n']})"
    s = make_problem(cfg)
    N, nnz = s.A.n_rows, s.A.nnz
    mdof = N / 1e6
    gpu = api.GpuOptions(device=local)
    comm = None
    if use_dist:   # one NCCL communicator for every hierarchy of the run
        nid = api.nccl_unique_id() if rank == 0 else bytes(128)
        if dist is not None:
            obj = [nid]
            dist.broadcast_object_list(obj, src=0)
            nid = obj[0]
        comm = api.NcclComm(nid, world, rank, local)

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

    # ---- inputs resident in HBM (value)
    d_rp = torch.from_numpy(s.A.row_ptr).to(dev)
    d_col = torch.from_numpy(s.A.col_idx).to(dev)
    d_val = torch.from_numpy(s.A.values).to(dev)
    d_xy = torch.from_numpy(np.ascontiguousarray(s.coords)).to(dev)
    d_b = torch.from_numpy(s.b).to(dev)
    d_u = torch.empty(N, dtype=torch.float64, device=dev)

    def device_step():
        h = setup_dev()
        r = api.solve_device(h, d_b.data_ptr(), d_u.data_ptr(), N)
        return h, r

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        h, r = device_step()
        del h
    barrier()
    launches0 = api.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    prof = {}
    iters = None
    setup_ms, solve_ms = [], []
    with ClockSampler(local) as clk:
        barrier()
        ev0.record()
        for k in range(args.steps):
            h = setup_dev()
            r = api.solve_device(h, d_b.data_ptr(), d_u.data_ptr(), N)
            iters = r.iterations
            a, b = h.last_timing()
            setup_ms.append(a)
            solve_ms.append(b)
            del h
        ev1.record()
        barrier()
    launches = api.launch_count() - launches0
    # one more (untimed) step with CUDA events around the finest-level kernels
    # on their launch stream: the roofline's per-launch kernel times
    h = setup_dev()
    h.profile(True)
    api.solve_device(h, d_b.data_ptr(), d_u.data_ptr(), N)
    for kind in PROFILE_KINDS:
        prof[kind] = h.profile_read(kind)
    del h
    elapsed = ev0.elapsed_time(ev1)
    if dist is not None:
        t = torch.tensor([elapsed], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
    ms_step = elapsed / args.steps
    # whole-job throughput: the global problem (all GPUs' DoFs) per step
    value = ms_step / mdof
    u_dev = d_u.cpu().numpy()

    # ---- e2e through the host-buffer C ABI, pinned memory
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
    A_h = api.CsrMatrix(N, N, pin(s.A.row_ptr), pin(s.A.col_idx), pin(s.A.values))
    xy_h, b_h = pin(s.coords), pin(s.b)
    u_h = pin(np.zeros(N))
    h2d = A_h.row_ptr.nbytes + A_h.col_idx.nbytes + A_h.values.nbytes + xy_h.nbytes + b_h.nbytes
    d2h = N * 8
    for _ in range(max(1, args.warmup // 2)):
        h = setup_host(A_h, xy_h)
        api.solve(A_h, b_h, h, out=u_h)
        del h
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        h = setup_host(A_h, xy_h)
        res = api.solve(A_h, b_h, h, out=u_h)
        del h
    e1.record()
    barrier()
    e2e_ms = e0.elapsed_time(e1) / args.steps
    if dist is not None:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    if use_dist:   # each part wrote the entries of the DoFs it owns
        hq = setup_dev()
        ids = api.part_dofs(hq)
        del hq
        assert np.array_equal(res.u[ids], u_dev[ids]), "host-API and device-API solutions differ"
    else:
        assert np.array_equal(res.u, u_dev), "host-API and device-API solutions differ"

    # ---- roofline of the dominant finest-level kernel (live CUDA events)
    peak, peak_src = peaks()
    kind = max(prof, key=lambda k: prof[k][1])
    n_l, tot_ms, bytes_l = prof[kind]
    achieved = bytes_l / (tot_ms / n_l * 1e-3) / 1e9 if n_l else 0.0
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            traffic = json.load(f).get(args.config, {}).get(str(kind))
    except Exception:
        pass
    shares = {PROFILE_KINDS[k]: round(prof[k][1] / (sum(solve_ms) / len(solve_ms)), 4) for k in prof}

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": "ms/MDOF", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["name"], "N": N, "nnz": nnz, "iterations": iters, "rtol": 1e-6,
                       "parallelism": (f"quadtree-subtree partition over {world} GPUs, NCCL halo/ghost exchange "
                                       "+ all-reduce, coarse levels agglomerated on rank 0") if use_dist else "1 GPU",
                       "setup_ms": statistics.median(setup_ms), "solve_ms": statistics.median(solve_ms),
                       "l2": f"inputs {(s.A.values.nbytes + s.A.col_idx.nbytes + 24 * N) / 1e6:.0f} MB > 126 MB L2"},
            "e2e": {"value": e2e_ms / mdof, "unit": "ms/MDOF", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h)},
            "roofline": {"bound": "hbm", "kernel": PROFILE_KINDS[kind], "achieved": achieved, "peak": peak,
                         "peak_source": peak_src, "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                         "launches": n_l, "algorithmic_bytes_per_launch": bytes_l,
                         "share_of_solve": shares},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        if world == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(cfg, s)
        print(json.dumps(out))
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

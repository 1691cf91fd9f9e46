"""Small setup + solve runs through every execution tier, for compute-sanitizer
(memcheck / racecheck / synccheck):  python tools/sanitize_cases.py [case ...]

Cases (each prints one line; exit code 1 if a solve fails to converge):
  tiles     jittered n=129: TMA tile kernels (fused tier capped at 64 cells)
  cluster   jittered n=129: 5-CTA cluster tier (DSMEM pushes) + single-CTA tier
  fused     jittered n=65: single-CTA tier only (TMA bulk staging, mbarrier)
  graded    graded n=65: finest block GS with large blocks (CTA / warp buckets)
  lu        jittered n=65, block_solve=1, coarse_solve=1 (reference-order LU paths)
  nograph   jittered n=65 with CUDA graphs off (eager launches, PDL chains)
  dist      jittered n=129 split over 2 parts on one device (in-process transport)
  c16       jittered n=257: the 128x128-cell level as 16-CTA clusters (cluster16.cu) + cluster tier
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1209_5421_b200 import api, problems  # noqa: E402


def run(name, s, g, dist_parts=0):
    if dist_parts:
        import threading
        res = [None] * dist_parts
        grp = api.LocalGroup(dist_parts)

        def part(p):
            h = api.setup_hierarchy_dist(s.A, s.coords, dist_parts, p, group=grp, gpu=g)
            res[p] = api.solve(s.A, s.b, h)
            del h
        th = [threading.Thread(target=part, args=(p,)) for p in range(dist_parts)]
        [t.start() for t in th]
        [t.join() for t in th]
        r = res[0]
    else:
        h = api.setup_hierarchy(s.A, s.coords, gpu=g)
        r = api.solve(s.A, s.b, h)
        r = api.solve(s.A, s.b, h)   # second solve: graph replay
        del h
    print(f"{name}: N={s.A.n_rows} iterations={r.iterations} converged={r.converged}", flush=True)
    return r.converged


CASES = {
    "tiles": lambda: run("tiles", problems.jittered_p1(129), api.GpuOptions(fused_max_cells=64, cluster_tier=False)),
    "cluster": lambda: run("cluster", problems.jittered_p1(129), api.GpuOptions(cluster_tier=True)),
    "fused": lambda: run("fused", problems.jittered_p1(65), api.GpuOptions()),
    "graded": lambda: run("graded", problems.graded_p1(65, 1.3), api.GpuOptions()),
    "lu": lambda: run("lu", problems.jittered_p1(65), api.GpuOptions(block_solve=1, coarse_solve=1)),
    "nograph": lambda: run("nograph", problems.jittered_p1(65), api.GpuOptions(use_graphs=False)),
    "dist": lambda: run("dist", problems.jittered_p1(129), api.GpuOptions(), dist_parts=2),
    "c16": lambda: run("c16", problems.jittered_p1(257), api.GpuOptions()),
}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    ok = all([CASES[n]() for n in names])
    sys.exit(0 if ok else 1)

"""Cluster tier on vs off (and vs the oracle) on a few problems:  python tools/cluster_check.py"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1209_5421_b200 import api, problems  # noqa: E402

cases = [("jitter257", problems.jittered_p1(257)), ("graded257", problems.graded_p1(257, 1.3)),
         ("p5_257", problems.poisson5(257)), ("jitter1025", problems.jittered_p1(1025)),
         ("graded2049", problems.graded_p1(2049, 1.3))]
for name, s in cases:
    out = {}
    for ct in (False, True):
        h = api.setup_hierarchy(s.A, s.coords, gpu=api.GpuOptions(cluster_tier=ct))
        r = api.solve(s.A, s.b, h)
        r2 = api.solve(s.A, s.b, h)
        out[ct] = (r, r2)
        del h
    a, b = out[False][0], out[True][0]
    d = np.max(np.abs(a.u - b.u)) / np.max(np.abs(a.u))
    det = np.array_equal(out[True][0].u, out[True][1].u)
    print(f"{name}: iters off {a.iterations} on {b.iterations}  rel diff {d:.2e}  deterministic {det}  "
          f"solve off {a.solve_seconds*1e3:.1f} ms on {out[True][1].solve_seconds*1e3:.1f} ms", flush=True)

"""One setup + a short solve for ncu captures:  python tools/prof_one.py graded2049 [max_outer]
(STREAM=<cells>: GpuOptions.stream_min_width; NOGRAPH=1: eager launches, so ncu sees the coarse kernels)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1209_5421_b200 import api, problems  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "graded2049"
max_outer = int(sys.argv[2]) if len(sys.argv) > 2 else 2
if name.startswith("jitter"):
    s = problems.jittered_p1(int(name[6:]))
elif name.startswith("graded"):
    s = problems.graded_p1(int(name[6:]), 1.3)
else:
    s = problems.poisson5(int(name[3:]))
h = api.setup_hierarchy(s.A, s.coords, gpu=api.GpuOptions(stream_min_width=int(os.environ.get("STREAM", "0")),
                                                          use_graphs=os.environ.get("NOGRAPH", "0") != "1"))
r = api.solve(s.A, s.b, h, api.CycleOptions(max_outer=max_outer))
print("iterations", r.iterations)

"""Host-API costs of the distributed path with one NCCL rank against the single-GPU path
(setup / solve / destroy wall times, C2):  python tools/dist_host_path.py"""
import os, sys, time
import numpy as np
sys.path.insert(0, os.getcwd())
from paper_1209_5421_b200 import api, problems
s = problems.graded_p1(2049, 1.3)
comm = api.NcclComm(api.nccl_unique_id(), 1, 0, 0)
for it in range(3):
    t0 = time.perf_counter()
    h = api.setup_hierarchy_dist(s.A, s.coords, 1, 0, comm=comm)
    t1 = time.perf_counter()
    r = api.solve(s.A, s.b, h)
    t2 = time.perf_counter()
    del h
    t3 = time.perf_counter()
    print(f"dist: setup {1e3*(t1-t0):.1f} ms solve {1e3*(t2-t1):.1f} ms (solve_seconds {1e3*r.solve_seconds:.1f}) destroy {1e3*(t3-t2):.1f} ms", flush=True)
for it in range(2):
    t0 = time.perf_counter()
    h = api.setup_hierarchy(s.A, s.coords)
    t1 = time.perf_counter()
    r = api.solve(s.A, s.b, h)
    t2 = time.perf_counter()
    del h
    t3 = time.perf_counter()
    print(f"single: setup {1e3*(t1-t0):.1f} ms solve {1e3*(t2-t1):.1f} ms destroy {1e3*(t3-t2):.1f} ms", flush=True)

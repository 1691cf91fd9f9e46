"""Multi-part path at C3 size on one GPU (in-process transport): correctness at
scale and the overhead of the distributed code path.  python tools/dist_scale.py [n] [parts]"""
import os
import sys
import time

import numpy as np
import scipy.sparse as sp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1209_5421_b200 import api, problems  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4097
parts = int(sys.argv[2]) if len(sys.argv) > 2 else 4
s = problems.jittered_p1(n)
A = sp.csr_matrix((s.A.values, s.A.col_idx, s.A.row_ptr), shape=(s.A.n_rows, s.A.n_rows))
for P in (1, parts):
    t0 = time.time()
    u, res, st = api.solve_parts(s.A, s.coords, s.b, P)
    t1 = time.time()
    rr = np.linalg.norm(s.b - A @ u) / np.linalg.norm(s.b)
    print(f"N={s.A.n_rows} parts={P}: iterations {res[0].iterations} converged {res[0].converged} "
          f"true rel residual {rr:.3e} opcx {st[0].operator_complexity:.4f} wall {t1 - t0:.1f}s "
          f"solve {res[0].solve_seconds:.3f}s", flush=True)

# launch overhead of the distributed code path with one rank: the single-GPU
# path, the NCCL transport (graph-captured coarse cycle) and the in-process one
h = api.setup_hierarchy(s.A, s.coords)
for _ in range(2):
    r = api.solve(s.A, s.b, h)
print(f"single-GPU path: iterations {r.iterations} solve {r.solve_seconds:.3f}s", flush=True)
del h
comm = api.NcclComm(api.nccl_unique_id(), 1, 0, 0)
h = api.setup_hierarchy_dist(s.A, s.coords, 1, 0, comm=comm)
for _ in range(2):
    r = api.solve(s.A, s.b, h)
print(f"dist path, NCCL 1 rank: iterations {r.iterations} solve {r.solve_seconds:.3f}s", flush=True)
del h
grp = api.LocalGroup(1)
h = api.setup_hierarchy_dist(s.A, s.coords, 1, 0, group=grp)
for _ in range(2):
    r = api.solve(s.A, s.b, h)
print(f"dist path, local 1 part: iterations {r.iterations} solve {r.solve_seconds:.3f}s", flush=True)

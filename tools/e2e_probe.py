"""Where does the host-buffer (e2e) path spend its time?  C2 workload."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1209_5421_b200 import api, problems  # noqa: E402

s = problems.jittered_p1(int(sys.argv[1][6:])) if len(sys.argv) > 1 and sys.argv[1].startswith("jitter") else problems.graded_p1(2049, 1.3)
N = s.A.n_rows
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
A_h = api.CsrMatrix(N, N, pin(s.A.row_ptr), pin(s.A.col_idx), pin(s.A.values))
xy_h, b_h, u_h = pin(s.coords), pin(s.b), pin(np.zeros(N))
dev = torch.device("cuda", 0)
d = [torch.from_numpy(x).to(dev) for x in (s.A.row_ptr, s.A.col_idx, s.A.values, np.ascontiguousarray(s.coords), s.b)]
du = torch.empty(N, dtype=torch.float64, device=dev)
nbytes = sum(x.nbytes for x in (A_h.row_ptr, A_h.col_idx, A_h.values, xy_h, b_h))
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tmp = [torch.from_numpy(x).to(dev, non_blocking=True) for x in (A_h.row_ptr, A_h.col_idx, A_h.values, xy_h, b_h)]
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    h = api.setup_hierarchy(A_h, xy_h)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    r = api.solve(A_h, b_h, h, out=u_h)
    t3 = time.perf_counter()
    del h
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    hd = api.setup_hierarchy_device(N, s.A.nnz, d[0].data_ptr(), d[1].data_ptr(), d[2].data_ptr(), d[3].data_ptr(), N)
    torch.cuda.synchronize()
    t5 = time.perf_counter()
    rd = api.solve_device(hd, d[4].data_ptr(), du.data_ptr(), N)
    torch.cuda.synchronize()
    t6 = time.perf_counter()
    del hd
    torch.cuda.synchronize()
    t7 = time.perf_counter()
    print(f"torch H2D {nbytes/1e6:.0f} MB: {1e3*(t1-t0):.1f} ms ({nbytes/(t1-t0)/1e9:.1f} GB/s) | host setup {1e3*(t2-t1):.1f} "
          f"solve {1e3*(t3-t2):.1f} destroy {1e3*(t4-t3):.1f} | device setup {1e3*(t5-t4):.1f} solve {1e3*(t6-t5):.1f} "
          f"destroy {1e3*(t7-t6):.1f}", flush=True)

"""Where does one bench step (device-resident inputs: setup_device + solve_device
+ destroy) spend its wall time?  python tools/step_probe.py [jitter4097]"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1209_5421_b200 import api, problems  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "jitter4097"
s = problems.jittered_p1(int(name[6:])) if name.startswith("jitter") else problems.graded_p1(int(name[6:]), 1.3)
N = s.A.n_rows
dev = torch.device("cuda", 0)
d = [torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in (s.A.row_ptr, s.A.col_idx, s.A.values, s.coords, s.b)]
du = torch.empty(N, dtype=torch.float64, device=dev)
for rep in range(6):
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    t0 = time.perf_counter()
    e[0].record()
    hd = api.setup_hierarchy_device(N, s.A.nnz, d[0].data_ptr(), d[1].data_ptr(), d[2].data_ptr(), d[3].data_ptr(), N)
    t1 = time.perf_counter()
    e[1].record()
    rd = api.solve_device(hd, d[4].data_ptr(), du.data_ptr(), N)
    t2 = time.perf_counter()
    e[2].record()
    a, b = hd.last_timing()
    del hd
    t3 = time.perf_counter()
    e[3].record()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print(f"host: setup {1e3*(t1-t0):.2f} solve {1e3*(t2-t1):.2f} destroy {1e3*(t3-t2):.2f} tail {1e3*(t4-t3):.2f} | "
          f"events: setup {e[0].elapsed_time(e[1]):.2f} solve {e[1].elapsed_time(e[2]):.2f} destroy {e[2].elapsed_time(e[3]):.2f} "
          f"total {e[0].elapsed_time(e[3]):.2f} | device setup {a:.2f} solve {b:.2f}", flush=True)

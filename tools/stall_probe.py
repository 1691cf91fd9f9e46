"""Which host-side part of a step stalls while nvidia-smi polls the GPU?
python tools/stall_probe.py [graded2049] [steps]   (runs nvidia-smi -lms 50 meanwhile)"""
import os
import subprocess
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1209_5421_b200 import api, problems  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "graded2049"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
s = problems.graded_p1(int(name[6:]), 1.3) if name.startswith("graded") else problems.jittered_p1(int(name[6:]))
N = s.A.n_rows
dev = torch.device("cuda", 0)
d = [torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in (s.A.row_ptr, s.A.col_idx, s.A.values, s.coords, s.b)]
du = torch.empty(N, dtype=torch.float64, device=dev)
for _ in range(3):
    h = api.setup_hierarchy_device(N, s.A.nnz, d[0].data_ptr(), d[1].data_ptr(), d[2].data_ptr(), d[3].data_ptr(), N)
    api.solve_device(h, d[4].data_ptr(), du.data_ptr(), N)
    del h
torch.cuda.synchronize()
q = os.environ.get("SMI_Q", "clocks.sm,clocks_event_reasons.active")
smi = None if q == "off" else subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader",
                                               "-lms", os.environ.get("SMI_MS", "50")],
                                              stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
time.sleep(float(os.environ.get("SMI_WAIT", "1.0")))
for k in range(steps):
    t0 = time.perf_counter()
    h = api.setup_hierarchy_device(N, s.A.nnz, d[0].data_ptr(), d[1].data_ptr(), d[2].data_ptr(), d[3].data_ptr(), N)
    t1 = time.perf_counter()
    api.solve_device(h, d[4].data_ptr(), du.data_ptr(), N)
    t2 = time.perf_counter()
    a, b = h.last_timing()
    del h
    t3 = time.perf_counter()
    print(f"step {k:2d}: host setup {1e3*(t1-t0):7.2f} (dev {a:6.2f})  solve {1e3*(t2-t1):7.2f} (dev {b:6.2f})  "
          f"destroy {1e3*(t3-t2):6.2f}", flush=True)
if smi is not None:
    smi.terminate()

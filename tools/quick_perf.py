"""Quick GPU timing probe (not the bench contract): setup + solve wall times
for a few BASELINE configurations through the C ABI."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1209_5421_b200 import api, problems  # noqa: E402

cfgs = sys.argv[1:] or ["jitter1025", "graded2049"]
for name in cfgs:
    t = time.time()
    if name.startswith("jitter"):
        s = problems.jittered_p1(int(name[6:]))
    elif name.startswith("graded"):
        s = problems.graded_p1(int(name[6:]), 1.3)
    elif name.startswith("p5_"):
        s = problems.poisson5(int(name[3:]))
    tg = time.time() - t
    for rep in range(3):
        t0 = time.time()
        h = api.setup_hierarchy(s.A, s.coords)
        t1 = time.time()
        r = api.solve(s.A, s.b, h)
        t2 = time.time()
        st = h.stats()
        print(f"{name}: N={s.A.n_rows} nnz={s.A.nnz} gen={tg:.2f}s setup={1e3*(t1-t0):.1f}ms "
              f"solve={1e3*(t2-t1):.1f}ms iters={r.iterations} conv={r.converged} levels={st.levels} "
              f"opcx={st.operator_complexity:.4f} ms/MDOF={1e3*(t2-t0)/(s.A.n_rows/1e6):.1f} "
              f"launches={api.launch_count()}", flush=True)
        del h

"""Quick GPU timing probe (not the bench contract): setup + solve times for a
few BASELINE configurations through the C ABI.  FUSED=<cells> sets
GpuOptions.fused_max_cells, CLUSTER=0 turns the cluster tier off, STREAM=<cells>
sets GpuOptions.stream_min_width (-1 off), C16=0 turns the 16-CTA cluster level off; AUX_TRACE=1 prints the device-time breakdown."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1209_5421_b200 import api, problems  # noqa: E402

cfgs = sys.argv[1:] or ["jitter1025", "graded2049"]
fused = int(os.environ.get("FUSED", "-1"))
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
        h = api.setup_hierarchy(s.A, s.coords, gpu=api.GpuOptions(fused_max_cells=fused, cluster_tier=os.environ.get("CLUSTER", "1") != "0",
                                                                  stream_min_width=int(os.environ.get("STREAM", "0")),
                                                                  cluster16=os.environ.get("C16", "1") != "0"))
        t1 = time.time()
        for k in range(2):
            ts = time.time()
            r = api.solve(s.A, s.b, h)
            te = time.time()
            st = h.stats()
            print(f"{name}: N={s.A.n_rows} gen={tg:.2f}s setup={1e3*(t1-t0):.1f}ms solve[{k}]={1e3*(te-ts):.1f}ms "
                  f"iters={r.iterations} conv={r.converged} levels={st.levels} opcx={st.operator_complexity:.4f} "
                  f"launches={api.launch_count()}", flush=True)
        del h

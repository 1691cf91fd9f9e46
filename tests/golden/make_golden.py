"""Regenerate tests/golden/golden.npz from the reference itself (oracle/_ref:
the unmodified reference headers compiled in place by oracle/Makefile).

    python tests/golden/make_golden.py

For each small problem of the BASELINE families the fixture stores what the
reference computes: level-L aggregation (agg_of), level sizes / nnz /
operator complexity, the level-L operator values, the coarsest LU, the
iteration count, the residual history and the solution.  tests/test_golden.py
checks the oracle (CPU) and the CUDA path (GPU) against these vectors, so
parity does not depend on /root/reference being present."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import bindings as ob  # noqa: E402
from paper_1209_5421_b200 import problems  # noqa: E402

CASES = {
    "poisson5_40": lambda: problems.poisson5(40),
    "jitter_48": lambda: problems.jittered_p1(48),
    "graded_64": lambda: problems.graded_p1(64, 1.3),
    "disk_40": lambda: problems.disk_p1(40),
    "jump_48": lambda: problems.jittered_p1(48, jump=1e3),
}


def main():
    out = {}
    for name, make in CASES.items():
        s = make()
        h = ob.CpuHierarchy("ref", s.A, s.coords)
        e = h.export()
        r = h.solve(s.b)
        out[f"{name}/agg_of"] = e["levels"][0]["agg_of"]
        out[f"{name}/sizes"] = np.array(e["stats"]["sizes"], np.int64)
        out[f"{name}/nnz"] = np.array(e["stats"]["nnz"], np.int64)
        out[f"{name}/opcx"] = np.array([e["stats"]["operator_complexity"]])
        out[f"{name}/ell_val_L"] = e["levels"][1]["ell_val"]
        out[f"{name}/coarsest_lu"] = e["coarsest_lu"]
        out[f"{name}/iterations"] = np.array([r["iterations"]])
        out[f"{name}/residual_history"] = r["residual_history"]
        out[f"{name}/u"] = r["u"]
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    print("wrote", os.path.join(HERE, "golden.npz"), len(out), "arrays")


if __name__ == "__main__":
    main()

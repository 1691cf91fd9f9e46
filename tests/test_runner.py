"""The batch runner with a backend switch (SURVEY 8(f) rank 3,
paper_1209_5421_b200/runner.py mirroring runner.hpp:87-197): the reference
backend runs here on CPU; the b200 backend must emit identical columns,
iteration counts and level statistics (GPU)."""
import io
import json

import pytest

from paper_1209_5421_b200 import runner


def test_reference_backend_csv_and_jsonl():
    reps = [runner.run_one("poisson2d", 33, backend="reference"), runner.run_one("jitter", 33, backend="reference")]
    out = io.StringIO()
    runner.write_csv(reps, out)
    lines = out.getvalue().splitlines()
    assert lines[0] == "N,levels,opcomplexity,iters,setup_s,solve_s,total_s,converged"
    assert lines[1].startswith("1024,") and lines[1].endswith(",1")
    js = io.StringIO()
    runner.write_jsonl(reps, js)
    d = json.loads(js.getvalue().splitlines()[0])
    assert d["label"] == "poisson2d-33" and d["n"] == 1024 and d["levels"] == len(d["level_sizes"])
    assert len(d["residual_history"]) == d["iters"] + 1
    res = io.StringIO()
    runner.write_residuals(reps, res)
    assert res.getvalue().splitlines()[0] == "N,iter,residual"


def test_cli_argument_error_exit_code(capsys):
    assert runner.main(["--gen", "poisson2d", "--n", "33", "--n-inner", "0", "--backend", "reference"]) == 1


@pytest.mark.gpu
@pytest.mark.parametrize("gpus", [1, 2])
def test_b200_backend_matches_reference_backend(gpus):
    for gen, n in (("poisson2d", 129), ("graded", 129)):
        ref = runner.run_one(gen, n, backend="reference")
        got = runner.run_one(gen, n, backend="b200", gpus=gpus)
        assert (got.n, got.nnz, got.levels, got.level_sizes, got.level_nnz) == \
               (ref.n, ref.nnz, ref.levels, ref.level_sizes, ref.level_nnz)
        assert round(got.opcomplexity, 4) == round(ref.opcomplexity, 4)
        assert abs(got.iters - ref.iters) <= 1 and got.converged == ref.converged

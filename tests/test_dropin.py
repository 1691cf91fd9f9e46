"""The C++ drop-in: tests/cpp/dropin.cpp calls the reference and the B200
library with the reference's own types, options and exception classes
(built by __graft_entry__.build() where the reference headers exist)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "dropin")


@pytest.mark.gpu
def test_cpp_dropin_parity():
    if not os.path.exists(BIN):
        pytest.skip("tests/cpp/dropin not built (needs the reference headers at build time)")
    p = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    print(p.stdout)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "dropin: OK" in p.stdout
    assert "caught auxamg::definiteness_error" in p.stdout


def test_cpp_header_compiles_without_reference(tmp_path):
    """auxamg_b200.hpp is self-contained (own error classes) when the
    reference headers are absent."""
    src = tmp_path / "t.cpp"
    src.write_text('#include "auxamg_b200.hpp"\n'
                   "struct Csr { int n_rows = 0, n_cols = 0; std::vector<int> row_ptr, col_idx; std::vector<double> values; };\n"
                   "struct P { double x, y; };\n"
                   "int main() { Csr a; std::vector<P> c; try { auto h = auxamg_b200::setup_hierarchy(a, c); }\n"
                   "  catch (const auxamg_b200::error&) {} return 0; }\n")
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", f"-I{os.path.join(ROOT, 'include')}", str(src)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr

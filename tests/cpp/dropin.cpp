// tests/cpp/dropin.cpp — the drop-in in C++: the same call sequence the
// reference runner makes (runner.hpp:99-105), once through the reference
// (header-only, CPU) and once through auxamg_b200.hpp (B200), on the
// reference's own problem generator and types.  Built by __graft_entry__.build()
// where the reference headers exist; the binary travels to the GPU box and is
// run by tests/test_dropin.py.  Exit 0 = parity (iterations +-1, u within 1e-12).
#include <algorithm>
#include <cmath>
#include <cstdio>

#include "auxamg/auxamg.hpp"
#include "auxamg_b200.hpp"

int main() {
    const auxamg::LinearSystem sys = auxamg::gen_poisson_uniform2d(129);
    auxamg::SetupOptions so;
    auxamg::CycleOptions co;

    const auxamg::Hierarchy href = auxamg::setup_hierarchy(sys.A, sys.coords, so);
    const auxamg::SolveResult rref = auxamg::solve(sys.A, sys.b, href, co);

    // the drop-in: same arguments, same option structs, same result fields
    const auxamg_b200::Hierarchy hgpu = auxamg_b200::setup_hierarchy(sys.A, sys.coords, so);
    const auxamg_b200::SolveResult rgpu = auxamg_b200::solve(sys.A, sys.b, hgpu, co);
    const auxamg::HierarchyStats sref = auxamg::stats(href);
    const auxamg_b200::HierarchyStats sgpu = auxamg_b200::stats(hgpu);

    double du = 0.0, um = 0.0;
    for (size_t i = 0; i < rref.u.size(); ++i) {
        du = std::max(du, std::abs(rgpu.u[i] - rref.u[i]));
        um = std::max(um, std::abs(rref.u[i]));
    }
    const double rel = du / um;
    std::printf("dropin: N=%d levels ref=%d gpu=%d opcx ref=%.6f gpu=%.6f iterations ref=%d gpu=%d max rel du=%.3e\n",
                sys.A.n_rows, sref.levels, sgpu.levels, sref.operator_complexity, sgpu.operator_complexity,
                rref.iterations, rgpu.iterations, rel);
    bool ok = std::abs(rref.iterations - rgpu.iterations) <= 1 && rel <= 1e-12 && sref.sizes == sgpu.sizes &&
              sref.nnz == sgpu.nnz && sref.operator_complexity == sgpu.operator_complexity;

    // the reference's exception classes come through unchanged
    auxamg::CsrMatrix bad = sys.A;
    bad.values[0] = -1.0;
    try {
        (void)auxamg_b200::setup_hierarchy(bad, sys.coords, so);
        ok = false;
    } catch (const auxamg::definiteness_error& e) {
        std::printf("dropin: caught auxamg::definiteness_error: %s\n", e.what());
    }
    std::printf("dropin: %s\n", ok ? "OK" : "FAIL");
    return ok ? 0 : 1;
}

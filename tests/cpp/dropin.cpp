// tests/cpp/dropin.cpp — the drop-in in C++: the same call sequence the
// reference runner makes (runner.hpp:99-105), once through the reference
// (header-only, CPU) and once through auxamg_b200.hpp (B200), on the
// reference's own problem generator and types.  Built by __graft_entry__.build()
// where the reference headers exist; the binary travels to the GPU box and is
// run by tests/test_dropin.py.  Exit 0 = parity (iterations +-1, u within 1e-12).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <utility>
#include <vector>

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

    auto compare = [&](const char* what, const auxamg::SolveResult& a, const auxamg_b200::SolveResult& b) {
        double d = 0.0, m = 0.0;
        for (size_t i = 0; i < a.u.size(); ++i) {
            d = std::max(d, std::abs(b.u[i] - a.u[i]));
            m = std::max(m, std::abs(a.u[i]));
        }
        const bool good = std::abs(a.iterations - b.iterations) <= 1 && d / m <= 1e-12;
        std::printf("dropin: %s iterations ref=%d gpu=%d max rel du=%.3e %s\n", what, a.iterations, b.iterations,
                    d / m, good ? "ok" : "MISMATCH");
        return good;
    };
    // solve() with a content-equal copy of A (cycle.hpp:202-208 checks only the order)
    {
        const auxamg::CsrMatrix A2 = sys.A;
        ok = compare("copied A", auxamg::solve(A2, sys.b, href, co), auxamg_b200::solve(A2, sys.b, hgpu, co)) && ok;
    }
    // solve() with a different A of the same order: the reference runs the
    // cycle on its setup copy and the outer A z on the caller's A (cycle.hpp:228)
    {
        auxamg::CsrMatrix A3 = sys.A;
        for (size_t p = 0; p < A3.values.size(); ++p) A3.values[p] *= (p % 7 == 0) ? 1.0001 : 1.0;
        ok = compare("values-modified A", auxamg::solve(A3, sys.b, href, co), auxamg_b200::solve(A3, sys.b, hgpu, co)) && ok;
        auxamg::CsrMatrix A4 = sys.A;   // a stored explicit zero in every row: another pattern
        auxamg::CsrMatrix A5;
        A5.n_rows = A4.n_rows;
        A5.n_cols = A4.n_cols;
        A5.row_ptr.push_back(0);
        for (int r = 0; r < A4.n_rows; ++r) {
            std::vector<std::pair<int, double>> row;
            bool has = false;
            for (int p = A4.row_ptr[r]; p < A4.row_ptr[r + 1]; ++p) {
                row.push_back({A4.col_idx[p], A4.values[p] * 1.5});
                has = has || A4.col_idx[p] == r + 2;
            }
            if (r + 2 < A4.n_rows && !has) row.push_back({r + 2, 0.0});
            std::sort(row.begin(), row.end());
            for (const auto& e : row) {
                A5.col_idx.push_back(e.first);
                A5.values.push_back(e.second);
            }
            A5.row_ptr.push_back(static_cast<int>(A5.col_idx.size()));
        }
        ok = compare("other-pattern A", auxamg::solve(A5, sys.b, href, co), auxamg_b200::solve(A5, sys.b, hgpu, co)) && ok;
    }
    // a different matrix at the setup matrix's own addresses (edited in place
    // everywhere, as after a free and reallocation): the sampled fingerprint
    // sees it and the outer A z uses the new values
    {
        auxamg::CsrMatrix A6 = sys.A;
        const auxamg_b200::Hierarchy h6 = auxamg_b200::setup_hierarchy(A6, sys.coords, so);
        const auxamg::Hierarchy r6 = auxamg::setup_hierarchy(A6, sys.coords, so);
        for (auto& v : A6.values) v *= 2.0;
        ok = compare("setup matrix rescaled in place", auxamg::solve(A6, sys.b, r6, co), auxamg_b200::solve(A6, sys.b, h6, co)) && ok;
    }

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

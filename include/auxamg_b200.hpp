// auxamg_b200.hpp — C++20 host API of the B200 auxiliary-grid AMG, a drop-in
// for the reference's setup + solve path:
//
//   auxamg::setup_hierarchy(A, coords, opts)   hierarchy.hpp:315-386
//   auxamg::solve(A, b, h, opts)               cycle.hpp:202-247
//   auxamg::stats(h)                           hierarchy.hpp:395-406
//   auxamg::set_num_threads(n)                 parallel.hpp:43-45
//
// Header-only over the C ABI (auxamg_b200.h).  The functions accept the
// reference's own types by shape: any CSR with n_rows / n_cols / row_ptr /
// col_idx / values (int32 / double vectors), any contiguous range of
// {double x, y} points, and any option struct with the reference's field
// names.  When the reference's errors.hpp is visible, failures are thrown as
// the reference's own exception classes (auxamg::size_error, ...), so existing
// catch blocks keep working; otherwise as auxamg_b200::* classes of the same
// names and hierarchy.
#pragma once

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "auxamg_b200.h"

#if __has_include("auxamg/errors.hpp")
#include "auxamg/errors.hpp"
#define AUXAMG_B200_REFERENCE_ERRORS 1
#endif

namespace auxamg_b200 {

#ifdef AUXAMG_B200_REFERENCE_ERRORS
using error = auxamg::error;
using size_error = auxamg::size_error;
using capacity_error = auxamg::capacity_error;
using structure_error = auxamg::structure_error;
using argument_error = auxamg::argument_error;
using geometry_error = auxamg::geometry_error;
using definiteness_error = auxamg::definiteness_error;
using singular_error = auxamg::singular_error;
using io_error = auxamg::io_error;
using parse_error = auxamg::parse_error;
#else
class error : public std::runtime_error { public: using std::runtime_error::runtime_error; };
class size_error : public error { public: using error::error; };
class capacity_error : public error { public: using error::error; };
class structure_error : public error { public: using error::error; };
class argument_error : public error { public: using error::error; };
class geometry_error : public error { public: using error::error; };
class definiteness_error : public error { public: using error::error; };
class singular_error : public error { public: using error::error; };
class io_error : public error { public: using error::error; };
class parse_error : public error {
public:
    parse_error(const std::string& what, long line)
        : error(what + " (line " + std::to_string(line) + ")"), line_(line) {}
    long line() const noexcept { return line_; }

private:
    long line_;
};
#endif
/// Device failure (no reference analogue).
class device_error : public error { public: using error::error; };

inline void throw_status(aux_status s, const char* msg) {
    const std::string m(msg);
    switch (s) {
        case AUX_OK: return;
        case AUX_SIZE_ERROR: throw size_error(m);
        case AUX_CAPACITY_ERROR: throw capacity_error(m);
        case AUX_STRUCTURE_ERROR: throw structure_error(m);
        case AUX_ARGUMENT_ERROR: throw argument_error(m);
        case AUX_GEOMETRY_ERROR: throw geometry_error(m);
        case AUX_DEFINITENESS_ERROR: throw definiteness_error(m);
        case AUX_SINGULAR_ERROR: throw singular_error(m);
        case AUX_IO_ERROR: throw io_error(m);
        case AUX_PARSE_ERROR: {   // what() ends in " (line N)" (errors.hpp:67-76)
            const size_t k = m.rfind(" (line ");
            if (k != std::string::npos && m.size() > k + 8 && m.back() == ')')
                throw parse_error(m.substr(0, k), std::stol(m.substr(k + 7, m.size() - k - 8)));
            throw parse_error(m, -1);
        }
        default: throw device_error(m);
    }
}

/// auxamg::SetupOptions (hierarchy.hpp:29-34), same fields and defaults.
struct SetupOptions {
    int coarsest_size = 64;
    bool strict_locality = false;
    bool lump_locality = false;
    double symmetry_tol = 1e-10;
};

/// auxamg::CycleOptions (cycle.hpp:30-37), same fields and defaults.
struct CycleOptions {
    int n_inner = 2;
    int pre_sweeps = 1;
    int post_sweeps = 1;
    int max_outer = 100;
    double rtol = 1e-6;
    int max_directions = 0;
};

/// auxamg::SolveResult (cycle.hpp:47-55).  Converts to any struct with the
/// reference's field names (e.g. auxamg::SolveResult itself), so a caller
/// written against the reference keeps its result types.
struct SolveResult {
    std::vector<double> u;
    std::vector<double> residual_history;
    int iterations = 0;
    bool converged = false;
    double setup_seconds = 0.0;
    double solve_seconds = 0.0;
    double total_seconds = 0.0;

    template <class T>
        requires requires(T t) { t.u; t.residual_history; t.iterations; t.converged; t.solve_seconds; }
    operator T() const {
        T t{};
        t.u = u;
        t.residual_history = residual_history;
        t.iterations = iterations;
        t.converged = converged;
        t.setup_seconds = setup_seconds;
        t.solve_seconds = solve_seconds;
        t.total_seconds = total_seconds;
        return t;
    }
};

/// auxamg::HierarchyStats (hierarchy.hpp:388-393); converts like SolveResult.
struct HierarchyStats {
    int levels = 0;
    std::vector<long> sizes;
    std::vector<long> nnz;
    double operator_complexity = 1.0;

    template <class T>
        requires requires(T t) { t.levels; t.sizes; t.nnz; t.operator_complexity; }
    operator T() const {
        T t{};
        t.levels = levels;
        t.sizes.assign(sizes.begin(), sizes.end());
        t.nnz.assign(nnz.begin(), nnz.end());
        t.operator_complexity = operator_complexity;
        return t;
    }
};

/// Device-resident auxamg::Hierarchy; move-only RAII owner of the GPU state.
class Hierarchy {
public:
    Hierarchy() = default;
    explicit Hierarchy(aux_hierarchy* h) : h_(h) {}
    Hierarchy(Hierarchy&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
    Hierarchy& operator=(Hierarchy&& o) noexcept {
        if (this != &o) { reset(); h_ = std::exchange(o.h_, nullptr); }
        return *this;
    }
    Hierarchy(const Hierarchy&) = delete;
    Hierarchy& operator=(const Hierarchy&) = delete;
    ~Hierarchy() { reset(); }
    int n_levels() const { return h_ ? aux_n_levels(h_) : 0; }
    aux_hierarchy* handle() const { return h_; }

private:
    void reset() {
        if (h_) aux_destroy(h_);
        h_ = nullptr;
    }
    aux_hierarchy* h_ = nullptr;
};

namespace detail {

template <class Csr>
aux_csr_view view(const Csr& A) {
    static_assert(sizeof(A.row_ptr[0]) == 4 && sizeof(A.col_idx[0]) == 4 && sizeof(A.values[0]) == 8,
                  "CSR must use int32 indices and double values (sparse.hpp:57-74)");
    aux_csr_view v;
    v.n_rows = A.n_rows;
    v.n_cols = A.n_cols;
    v.nnz = static_cast<int64_t>(A.values.size());
    v.row_ptr = reinterpret_cast<const int32_t*>(A.row_ptr.data());
    v.col_idx = reinterpret_cast<const int32_t*>(A.col_idx.data());
    v.values = A.values.data();
    return v;
}

template <class O>
aux_setup_opts setup_opts(const O& o) {
    aux_setup_opts c;
    c.coarsest_size = o.coarsest_size;
    c.strict_locality = o.strict_locality ? 1 : 0;
    c.lump_locality = o.lump_locality ? 1 : 0;
    c.symmetry_tol = o.symmetry_tol;
    return c;
}

template <class O>
aux_cycle_opts cycle_opts(const O& o) {
    aux_cycle_opts c;
    c.n_inner = o.n_inner;
    c.pre_sweeps = o.pre_sweeps;
    c.post_sweeps = o.post_sweeps;
    c.max_outer = o.max_outer;
    c.rtol = o.rtol;
    c.max_directions = o.max_directions;
    return c;
}

}  // namespace detail

/// setup_hierarchy(A, coords, opts) — hierarchy.hpp:315-386.  `coords` is any
/// contiguous range of 16-byte {double x, y} points (std::span<const Point>).
template <class Csr, class Points, class Opts = SetupOptions>
Hierarchy setup_hierarchy(const Csr& A, const Points& coords, const Opts& opts = Opts{},
                          const aux_gpu_opts* gpu = nullptr) {
    static_assert(sizeof(*std::data(coords)) == 2 * sizeof(double), "points must be {double x, y}");
    const aux_csr_view v = detail::view(A);
    const aux_setup_opts o = detail::setup_opts(opts);
    aux_hierarchy* h = nullptr;
    char msg[512];
    throw_status(aux_setup(&v, reinterpret_cast<const double*>(std::data(coords)),
                           static_cast<int64_t>(std::size(coords)), &o, gpu, &h, msg, sizeof msg),
                 msg);
    return Hierarchy(h);
}

/// solve(A, b, h, opts) — cycle.hpp:202-247.  As in the reference the cycle
/// runs on the hierarchy's copy of the setup matrix and the outer A z on the
/// caller's A: the setup matrix (same arrays, same sampled contents) reuses its
/// device copy, any other matrix of the same order is uploaded for that solve.
template <class Csr, class Opts = CycleOptions>
SolveResult solve(const Csr& A, std::span<const double> b, const Hierarchy& h, const Opts& opts = Opts{}) {
    const aux_csr_view v = detail::view(A);
    const aux_cycle_opts o = detail::cycle_opts(opts);
    SolveResult r;
    r.u.assign(static_cast<size_t>(A.n_rows), 0.0);
    r.residual_history.assign(static_cast<size_t>(std::max(o.max_outer, 0)) + 1, 0.0);   // options checked by aux_solve
    aux_solve_result res{};
    res.u = r.u.data();
    res.residual_history = r.residual_history.data();
    res.history_capacity = static_cast<int32_t>(r.residual_history.size());
    char msg[512];
    throw_status(aux_solve(h.handle(), &v, b.data(), static_cast<int64_t>(b.size()), &o, &res, msg, sizeof msg),
                 msg);
    r.residual_history.resize(static_cast<size_t>(res.history_len));
    r.iterations = res.iterations;
    r.converged = res.converged != 0;
    r.setup_seconds = res.setup_seconds;
    r.solve_seconds = res.solve_seconds;
    r.total_seconds = res.total_seconds;
    return r;
}

/// stats(h) — hierarchy.hpp:395-406.
inline HierarchyStats stats(const Hierarchy& h) {
    aux_stats_out s;
    throw_status(aux_stats(h.handle(), &s), "stats");
    HierarchyStats out;
    out.levels = s.levels;
    for (int i = 0; i < s.levels; ++i) {
        out.sizes.push_back(static_cast<long>(s.sizes[i]));
        out.nnz.push_back(static_cast<long>(s.nnz[i]));
    }
    out.operator_complexity = s.operator_complexity;
    return out;
}

/// set_num_threads(n) — parallel.hpp:43-45; accepted, no effect on the GPU path.
inline void set_num_threads(int n) { aux_set_num_threads(n); }

/// read_matrix_market(path) — matrix_market.hpp:33-104, multithreaded parse;
/// Csr is any CSR type with the reference's fields (auxamg::CsrMatrix).
template <class Csr>
Csr read_matrix_market(const std::string& path, int threads = 0) {
    aux_file_data* d = nullptr;
    char msg[512];
    throw_status(aux_read_matrix_market(path.c_str(), threads, &d, msg, sizeof msg), msg);
    int64_t n = 0, m = 0, nnz = 0;
    aux_file_data_sizes(d, &n, &m, &nnz);
    Csr A{};
    A.n_rows = static_cast<int>(n);
    A.n_cols = static_cast<int>(m);
    A.row_ptr.resize(static_cast<size_t>(n) + 1);
    A.col_idx.resize(static_cast<size_t>(nnz));
    A.values.resize(static_cast<size_t>(nnz));
    aux_file_data_copy(d, A.row_ptr.data(), A.col_idx.data(), A.values.data());
    aux_file_data_destroy(d);
    return A;
}

/// read_coords(path) — problems.hpp:313-330; Point is any {double x, y}.
template <class Point>
std::vector<Point> read_coords(const std::string& path, int threads = 0) {
    static_assert(sizeof(Point) == 2 * sizeof(double), "points must be {double x, y}");
    aux_file_data* d = nullptr;
    char msg[512];
    throw_status(aux_read_coords(path.c_str(), threads, &d, msg, sizeof msg), msg);
    int64_t n = 0;
    aux_file_data_sizes(d, &n, nullptr, nullptr);
    std::vector<Point> pts(static_cast<size_t>(n));
    aux_file_data_copy(d, pts.data(), nullptr, nullptr);
    aux_file_data_destroy(d);
    return pts;
}

}  // namespace auxamg_b200

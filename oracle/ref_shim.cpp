// oracle/ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// Exposes the UNMODIFIED reference library (/root/reference/proj/include/auxamg,
// header-only C++20) through the same plain C ABI as oracle/auxamg_oracle.c
// (ref_ prefix), so tests can pin the C restatement against the reference
// itself and bench.py can time the reference's own CPU path.  Built by
// oracle/Makefile into oracle/_ref/libauxamg_ref.so (git-ignored; the .so
// travels to the GPU box, the reference sources do not).
#include <cstring>
#include <exception>
#include <span>
#include <string>
#include <vector>

#include "auxamg/auxamg.hpp"
#include "auxamg/problems.hpp"
#include "testgen.hpp"   // reference tests/testgen.hpp (graded_mesh, disk_mesh, random_*)
#include "../include/auxamg_b200.h"

namespace {

struct RefH {
    auxamg::Hierarchy h;
};

template <class F>
int guarded(char* msg, size_t len, F&& f) {
    auto put = [&](const std::exception& ex) {
        if (msg && len) std::snprintf(msg, len, "%s", ex.what());
    };
    try {
        f();
        return AUX_OK;
    } catch (const auxamg::size_error& e) { put(e); return AUX_SIZE_ERROR; }
    catch (const auxamg::capacity_error& e) { put(e); return AUX_CAPACITY_ERROR; }
    catch (const auxamg::structure_error& e) { put(e); return AUX_STRUCTURE_ERROR; }
    catch (const auxamg::argument_error& e) { put(e); return AUX_ARGUMENT_ERROR; }
    catch (const auxamg::geometry_error& e) { put(e); return AUX_GEOMETRY_ERROR; }
    catch (const auxamg::definiteness_error& e) { put(e); return AUX_DEFINITENESS_ERROR; }
    catch (const auxamg::singular_error& e) { put(e); return AUX_SINGULAR_ERROR; }
    catch (const auxamg::io_error& e) { put(e); return AUX_IO_ERROR; }
    catch (const auxamg::parse_error& e) { put(e); return AUX_PARSE_ERROR; }
    catch (const std::exception& e) { put(e); return AUX_INTERNAL_ERROR; }
}

auxamg::CsrMatrix to_csr(const aux_csr_view* v) {
    auxamg::CsrMatrix A;
    A.n_rows = v->n_rows;
    A.n_cols = v->n_cols;
    A.row_ptr.assign(v->row_ptr, v->row_ptr + v->n_rows + 1);
    A.col_idx.assign(v->col_idx, v->col_idx + v->nnz);
    A.values.assign(v->values, v->values + v->nnz);
    return A;
}

// One generated input: the reference's own generators (problems.hpp,
// tests/testgen.hpp), so the harness generator libauxgen.so can be pinned
// byte for byte and the reference arm of bench.py maps no repo library.
struct RefGen {
    auxamg::LinearSystem sys;
    auxamg::TriMesh mesh;
    std::vector<double> xy;
    std::vector<int> ell_col;
    std::vector<double> ell_val;
};

// assemble_fem_triangle (problems.hpp:152-193) with the BASELINE C4 jump
// coefficient: the reference has no coefficient argument, so
// the element loop is restated around the reference's own element_geometry and
// csr_from_triplets, kappa multiplied before the division by 4*area.
auxamg::LinearSystem assemble_jump(const auxamg::TriMesh& mesh, double kappa_odd) {
    const int n = static_cast<int>(mesh.nodes.size());
    std::vector<char> is_boundary(n, 0);
    for (int v : mesh.boundary_nodes) is_boundary[v] = 1;
    std::vector<int> interior_of(n, -1);
    int n_interior = 0;
    for (int v = 0; v < n; ++v)
        if (!is_boundary[v]) interior_of[v] = n_interior++;
    auxamg::LinearSystem sys;
    sys.b.assign(n_interior, 0.0);
    sys.coords.resize(n_interior);
    for (int v = 0; v < n; ++v)
        if (interior_of[v] >= 0) sys.coords[interior_of[v]] = mesh.nodes[v];
    std::vector<auxamg::Triplet> entries;
    entries.reserve(mesh.triangles.size() * 9);
    for (int e = 0; e < static_cast<int>(mesh.triangles.size()); ++e) {
        const auto g = auxamg::detail::element_geometry(mesh, e);
        const auto& t = mesh.triangles[e];
        const auxamg::Point p0 = mesh.nodes[t[0]], p1 = mesh.nodes[t[1]], p2 = mesh.nodes[t[2]];
        const double cx = (p0.x + p1.x + p2.x) / 3.0, cy = (p0.y + p1.y + p2.y) / 3.0;
        const int bx = std::min(7, static_cast<int>(8.0 * cx)), by = std::min(7, static_cast<int>(8.0 * cy));
        const double kappa = ((bx + by) % 2 == 1) ? kappa_odd : 1.0;
        for (int a = 0; a < 3; ++a) {
            const int row = interior_of[t[a]];
            if (row < 0) continue;
            sys.b[row] += 1.0 * g.area / 3.0;
            for (int b = 0; b < 3; ++b) {
                const int col = interior_of[t[b]];
                if (col < 0) continue;
                entries.push_back({row, col, (kappa * (g.b[a] * g.b[b] + g.c[a] * g.c[b])) / (4.0 * g.area)});
            }
        }
    }
    sys.A = auxamg::csr_from_triplets(n_interior, n_interior, std::move(entries));
    return sys;
}

}  // namespace

extern "C" {

// Same kind numbering as libauxgen's auxgen_make (paper_1209_5421_b200/csrc/problems.cpp):
//   0 gen_poisson_uniform2d(n)                       problems.hpp:41-76
//   1 structured_split_mesh(n) + assemble             problems.hpp:80-105, 152-193
//   2 split mesh, interior nodes jittered by mt19937(seed) U(-param,param)*h
//   3 testgen::graded_mesh(n, param)                   tests/testgen.hpp:91-98
//   4 testgen::disk_mesh(n, 0.5, 0.5, param or 0.48)   tests/testgen.hpp:132-158
// jump > 0: the C4 checkerboard coefficient (kinds 1-4).
void* ref_gen_make(int kind, int n, double param, unsigned seed, double jump) {
    auto* g = new RefGen;
    try {
        if (kind == 0) {
            g->sys = auxamg::gen_poisson_uniform2d(n);
        } else {
            if (kind == 1 || kind == 2) g->mesh = auxamg::structured_split_mesh(n);
            if (kind == 2) {
                std::mt19937 rng(seed);
                std::uniform_real_distribution<double> U(-param, param);
                const double h = 1.0 / n;
                for (int j = 1; j < n; ++j)
                    for (int i = 1; i < n; ++i) {
                        auxamg::Point& p = g->mesh.nodes[static_cast<std::size_t>(j) * (n + 1) + i];
                        p.x += U(rng) * h;
                        p.y += U(rng) * h;
                    }
            } else if (kind == 3) {
                g->mesh = testgen::graded_mesh(n, param);
            } else if (kind == 4) {
                g->mesh = testgen::disk_mesh(n, 0.5, 0.5, param > 0 ? param : 0.48);
            } else if (kind != 1) {
                throw std::invalid_argument("unknown kind");
            }
            g->sys = jump > 0.0 ? assemble_jump(g->mesh, jump) : auxamg::assemble_fem_triangle(g->mesh, 1.0);
        }
        g->xy.resize(2 * g->sys.coords.size());
        for (std::size_t i = 0; i < g->sys.coords.size(); ++i) {
            g->xy[2 * i] = g->sys.coords[i].x;
            g->xy[2 * i + 1] = g->sys.coords[i].y;
        }
    } catch (...) {
        delete g;
        return nullptr;
    }
    return g;
}

// testgen::random_spd (tests/testgen.hpp:18-35)
void* ref_gen_random_spd(int n, unsigned seed) {
    auto* g = new RefGen;
    g->sys.A = testgen::random_spd(n, seed);
    return g;
}

// testgen::random_stencil (tests/testgen.hpp:39-61)
void* ref_gen_random_stencil(int k, unsigned seed) {
    auto* g = new RefGen;
    const auxamg::EllMatrix a = testgen::random_stencil(k, seed);
    g->ell_col = a.col_idx;
    g->ell_val = a.values;
    return g;
}

// testgen::random_vector (tests/testgen.hpp:79-86)
void ref_gen_random_vector(int64_t n, unsigned seed, double lo, double hi, double* out) {
    const std::vector<double> v = testgen::random_vector(static_cast<std::size_t>(n), seed, lo, hi);
    std::memcpy(out, v.data(), sizeof(double) * v.size());
}

int ref_gen_n(void* p) { return static_cast<RefGen*>(p)->sys.A.n_rows; }
int64_t ref_gen_nnz(void* p) { return static_cast<int64_t>(static_cast<RefGen*>(p)->sys.A.values.size()); }
const int* ref_gen_row_ptr(void* p) { return static_cast<RefGen*>(p)->sys.A.row_ptr.data(); }
const int* ref_gen_col_idx(void* p) { return static_cast<RefGen*>(p)->sys.A.col_idx.data(); }
const double* ref_gen_values(void* p) { return static_cast<RefGen*>(p)->sys.A.values.data(); }
const double* ref_gen_b(void* p) { return static_cast<RefGen*>(p)->sys.b.data(); }
const double* ref_gen_xy(void* p) { return static_cast<RefGen*>(p)->xy.data(); }
int64_t ref_gen_ell_len(void* p) { return static_cast<int64_t>(static_cast<RefGen*>(p)->ell_val.size()); }
const int* ref_gen_ell_col(void* p) { return static_cast<RefGen*>(p)->ell_col.data(); }
const double* ref_gen_ell_val(void* p) { return static_cast<RefGen*>(p)->ell_val.data(); }
int ref_gen_mesh_nodes(void* p) { return static_cast<int>(static_cast<RefGen*>(p)->mesh.nodes.size()); }
int ref_gen_mesh_tris(void* p) { return static_cast<int>(static_cast<RefGen*>(p)->mesh.triangles.size()); }
int ref_gen_mesh_nboundary(void* p) { return static_cast<int>(static_cast<RefGen*>(p)->mesh.boundary_nodes.size()); }
void ref_gen_mesh_copy(void* p, double* xy, int* tris, int* boundary) {
    const auxamg::TriMesh& m = static_cast<RefGen*>(p)->mesh;
    for (std::size_t i = 0; i < m.nodes.size(); ++i) { xy[2 * i] = m.nodes[i].x; xy[2 * i + 1] = m.nodes[i].y; }
    for (std::size_t i = 0; i < m.triangles.size(); ++i)
        for (int v = 0; v < 3; ++v) tris[3 * i + v] = m.triangles[i][v];
    for (std::size_t i = 0; i < m.boundary_nodes.size(); ++i) boundary[i] = m.boundary_nodes[i];
}
void ref_gen_free(void* p) { delete static_cast<RefGen*>(p); }

void ref_set_num_threads(int n) { auxamg::set_num_threads(n); }

int ref_setup(const aux_csr_view* Av, const double* xy, int64_t n_points, const aux_setup_opts* o,
              void** out, char* msg, size_t len) {
    *out = nullptr;
    return guarded(msg, len, [&] {
        auxamg::CsrMatrix A = to_csr(Av);
        std::vector<auxamg::Point> pts(static_cast<std::size_t>(n_points));
        for (int64_t i = 0; i < n_points; ++i) pts[i] = {xy[2 * i], xy[2 * i + 1]};
        auxamg::SetupOptions so;
        so.coarsest_size = o->coarsest_size;
        so.strict_locality = o->strict_locality != 0;
        so.lump_locality = o->lump_locality != 0;
        so.symmetry_tol = o->symmetry_tol;
        auto* r = new RefH{auxamg::setup_hierarchy(A, pts, so)};
        *out = r;
    });
}

void ref_destroy(void* h) { delete static_cast<RefH*>(h); }

int ref_solve(void* hp, const aux_csr_view* Av, const double* b, int64_t n_b, const aux_cycle_opts* o,
              aux_solve_result* res, char* msg, size_t len) {
    auto* H = static_cast<RefH*>(hp);
    return guarded(msg, len, [&] {
        auxamg::CycleOptions co;
        co.n_inner = o->n_inner;
        co.pre_sweeps = o->pre_sweeps;
        co.post_sweeps = o->post_sweeps;
        co.max_outer = o->max_outer;
        co.rtol = o->rtol;
        co.max_directions = o->max_directions;
        std::span<const double> bs(b, static_cast<std::size_t>(n_b));
        auxamg::SolveResult r;
        if (Av) {
            const auxamg::CsrMatrix A = to_csr(Av);
            r = auxamg::solve(A, bs, H->h, co);
        } else {
            r = auxamg::solve(H->h.levels.front().csr, bs, H->h, co);
        }
        if (res->u) std::memcpy(res->u, r.u.data(), r.u.size() * sizeof(double));
        res->history_len = static_cast<int32_t>(r.residual_history.size());
        for (std::size_t i = 0; i < r.residual_history.size() && static_cast<int>(i) < res->history_capacity; ++i)
            res->residual_history[i] = r.residual_history[i];
        res->iterations = r.iterations;
        res->converged = r.converged ? 1 : 0;
        res->setup_seconds = r.setup_seconds;
        res->solve_seconds = r.solve_seconds;
        res->total_seconds = r.total_seconds;
    });
}

int ref_n_levels(void* hp) { return static_cast<RefH*>(hp)->h.n_levels(); }

int ref_grid(void* hp, double box[4], int32_t* depth) {
    const auto& g = static_cast<RefH*>(hp)->h.grid;
    box[0] = g.a1; box[1] = g.b1; box[2] = g.a2; box[3] = g.b2;
    *depth = g.depth;
    return AUX_OK;
}

int ref_locality(void* hp, aux_locality* out) {
    const auto& l = static_cast<RefH*>(hp)->h.locality;
    out->dropped = l.dropped; out->dropped_mass = l.dropped_mass;
    out->lumped = l.lumped; out->lumped_mass = l.lumped_mass;
    return AUX_OK;
}

int ref_stats(void* hp, aux_stats_out* s) {
    const auxamg::HierarchyStats st = auxamg::stats(static_cast<RefH*>(hp)->h);
    s->levels = st.levels;
    for (int i = 0; i < st.levels && i < AUX_MAX_LEVELS; ++i) { s->sizes[i] = st.sizes[i]; s->nnz[i] = st.nnz[i]; }
    s->operator_complexity = st.operator_complexity;
    return AUX_OK;
}

int ref_level_info_get(void* hp, int32_t l, aux_level_info* o) {
    const auto& h = static_cast<RefH*>(hp)->h;
    if (l < 0 || l >= h.n_levels()) return AUX_ARGUMENT_ERROR;
    const auxamg::Level& lv = h.levels[l];
    std::memset(o, 0, sizeof *o);
    o->k = lv.k; o->structured = lv.structured; o->n = lv.n; o->nnz = lv.nnz;
    o->has_map = lv.to_coarser.agg_of.empty() ? 0 : 1;
    o->map_level = lv.to_coarser.level;
    o->n_aggregates = lv.to_coarser.n_aggregates;
    o->n_items = lv.schedule.n_items();
    long pool = 0;
    for (int s : lv.blocks.block_size) pool += static_cast<long>(s) * s;
    o->block_pool = pool;
    return AUX_OK;
}

int ref_export_level(void* hp, int32_t l, aux_level_export* x) {
    const auto& h = static_cast<RefH*>(hp)->h;
    if (l < 0 || l >= h.n_levels()) return AUX_ARGUMENT_ERROR;
    const auxamg::Level& lv = h.levels[l];
    const auto& m = lv.to_coarser;
    if (!m.agg_of.empty()) {
        if (x->agg_of) std::memcpy(x->agg_of, m.agg_of.data(), 4 * m.agg_of.size());
        if (x->member_ptr) std::memcpy(x->member_ptr, m.member_ptr.data(), 4 * m.member_ptr.size());
        if (x->member_idx) std::memcpy(x->member_idx, m.member_idx.data(), 4 * m.member_idx.size());
    }
    if (x->active) std::memcpy(x->active, lv.active.data(), lv.active.size());
    if (x->item_color && !lv.schedule.item_color.empty())
        std::memcpy(x->item_color, lv.schedule.item_color.data(), 4 * lv.schedule.item_color.size());
    if (lv.structured) {
        if (x->ell_col) std::memcpy(x->ell_col, lv.ell.col_idx.data(), 4 * lv.ell.col_idx.size());
        if (x->ell_val) std::memcpy(x->ell_val, lv.ell.values.data(), 8 * lv.ell.values.size());
    }
    if (!lv.blocks.block_size.empty()) {
        long off = 0, poff = 0;
        const int nb = static_cast<int>(lv.blocks.block_size.size());
        for (int g = 0; g < nb; ++g) {
            const int s = lv.blocks.block_size[g];
            if (x->block_size) x->block_size[g] = s;
            if (x->block_offset) x->block_offset[g] = off;
            if (s && x->block_lu) std::memcpy(x->block_lu + off, lv.blocks.factors[g].lu.data.data(), 8 * static_cast<size_t>(s) * s);
            if (s && x->block_perm) std::memcpy(x->block_perm + poff, lv.blocks.factors[g].perm.data(), 4 * static_cast<size_t>(s));
            off += static_cast<long>(s) * s;
            poff += s;
        }
        if (x->block_offset) x->block_offset[nb] = off;
    }
    return AUX_OK;
}

int ref_export_coarsest(void* hp, int32_t* n, double* lu, int32_t* perm) {
    const auto& c = static_cast<RefH*>(hp)->h.coarsest;
    *n = c.lu.n_rows;
    if (lu) std::memcpy(lu, c.lu.data.data(), 8 * c.lu.data.size());
    if (perm) std::memcpy(perm, c.perm.data(), 4 * c.perm.size());
    return AUX_OK;
}

// Kernel-level hooks used by the KAT tests.
int ref_choose_depth(long n, int* depth) {
    char m[8];
    return guarded(m, sizeof m, [&] { *depth = auxamg::choose_depth(n); });
}

int ref_subregion_of_point(double x, double y, const double box[4], int k, int* cell) {
    char m[8];
    return guarded(m, sizeof m, [&] {
        auxamg::AuxGrid g;
        g.a1 = box[0]; g.b1 = box[1]; g.a2 = box[2]; g.b2 = box[3];
        g.depth = k;
        *cell = auxamg::subregion_of_point(x, y, g, k);
    });
}

int ref_point_gs_sweep_ell(int k, const int* col, const double* val, const double* b, double* x, int dir,
                           char* msg, size_t len) {
    return guarded(msg, len, [&] {
        const int n = 1 << (2 * k);
        auxamg::EllMatrix A(n, 9);
        A.col_idx.assign(col, col + 9 * n);
        A.values.assign(val, val + 9 * n);
        const auxamg::ColorSchedule s = auxamg::make_schedule(k, std::vector<std::uint8_t>(n, 1));
        std::span<const double> bs(b, n);
        std::span<double> xs(x, n);
        auxamg::point_gs_sweep(A, bs, xs, s, dir == 0 ? auxamg::SweepDirection::forward
                                                      : auxamg::SweepDirection::transposed);
    });
}

double ref_dot(const double* a, const double* b, int64_t n) {
    return auxamg::dot(std::span<const double>(a, n), std::span<const double>(b, n));
}

// auxamg::galerkin_dense (hierarchy.hpp:239-247) on an arbitrary partition
int ref_galerkin_dense(const aux_csr_view* Av, const int32_t* agg_of, int64_t n_agg_of, int32_t n_agg, double* C) {
    return guarded(nullptr, 0, [&] {
        const auxamg::CsrMatrix A = to_csr(Av);
        auxamg::AggregationMap agg;
        agg.n_aggregates = n_agg;
        agg.agg_of.assign(agg_of, agg_of + n_agg_of);
        const auxamg::DenseMatrix D = auxamg::galerkin_dense(A, agg);
        for (int r = 0; r < n_agg; ++r)
            for (int c = 0; c < n_agg; ++c) C[(size_t)r * n_agg + c] = D(r, c);
    });
}

// ---- the reference's file readers (matrix_market.hpp:33-120, problems.hpp:201-330):
// results in a RefGen (CSR in sys.A, mesh in mesh, points in xy)
int ref_read_matrix_market(const char* path, void** out, char* msg, size_t len) {
    *out = nullptr;
    auto* g = new RefGen;
    const int st = guarded(msg, len, [&] { g->sys.A = auxamg::read_matrix_market(path); });
    if (st != AUX_OK) delete g;
    else *out = g;
    return st;
}
int ref_gen_ncols(void* p) { return static_cast<RefGen*>(p)->sys.A.n_cols; }
int ref_read_mesh(const char* path, void** out, char* msg, size_t len) {
    *out = nullptr;
    auto* g = new RefGen;
    const int st = guarded(msg, len, [&] { g->mesh = auxamg::read_mesh(path); });
    if (st != AUX_OK) delete g;
    else *out = g;
    return st;
}
int ref_read_coords(const char* path, void** out, int64_t* n, char* msg, size_t len) {
    *out = nullptr;
    auto* g = new RefGen;
    const int st = guarded(msg, len, [&] {
        const std::vector<auxamg::Point> pts = auxamg::read_coords(path);
        g->xy.resize(2 * pts.size());
        for (std::size_t i = 0; i < pts.size(); ++i) {
            g->xy[2 * i] = pts[i].x;
            g->xy[2 * i + 1] = pts[i].y;
        }
        *n = (int64_t)pts.size();
    });
    if (st != AUX_OK) delete g;
    else *out = g;
    return st;
}
// assemble_fem_triangle (problems.hpp:152-193, f = 1) of a given mesh
void* ref_assemble_mesh(const double* xy, int n_nodes, const int* tris, int n_tris, const int* bnd, int n_bnd) {
    auto* g = new RefGen;
    try {
        g->mesh.nodes.resize(n_nodes);
        for (int i = 0; i < n_nodes; ++i) g->mesh.nodes[i] = {xy[2 * i], xy[2 * i + 1]};
        g->mesh.triangles.resize(n_tris);
        for (int e = 0; e < n_tris; ++e) g->mesh.triangles[e] = {tris[3 * e], tris[3 * e + 1], tris[3 * e + 2]};
        g->mesh.boundary_nodes.assign(bnd, bnd + n_bnd);
        g->sys = auxamg::assemble_fem_triangle(g->mesh, 1.0);
        g->xy.resize(2 * g->sys.coords.size());
        for (std::size_t i = 0; i < g->sys.coords.size(); ++i) {
            g->xy[2 * i] = g->sys.coords[i].x;
            g->xy[2 * i + 1] = g->sys.coords[i].y;
        }
    } catch (...) {
        delete g;
        return nullptr;
    }
    return g;
}

int ref_write_matrix_market(const aux_csr_view* Av, const char* path, char* msg, size_t len) {
    return guarded(msg, len, [&] { auxamg::write_matrix_market(to_csr(Av), path); });
}

}  // extern "C"

// problems.cpp — synthetic input generators for the bench and the parity tests
// (harness code, not on the setup/solve path).  They reproduce the reference's
// problem sources so both the CUDA path and the oracle see byte-identical
// CSR/coordinates/right-hand sides:
//
//   gen_poisson_uniform2d           problems.hpp:41-76
//   structured_split_mesh           problems.hpp:80-105
//   element_geometry                problems.hpp:115-128
//   assemble_fem_triangle           problems.hpp:152-193  (optional jump coefficient)
//   csr_from_triplets               sparse.hpp:193-215   (std::sort, same comparator)
//   graded_mesh / disk_mesh         tests/testgen.hpp:91-98, 132-158
//   random_spd / random_stencil / random_vector   tests/testgen.hpp:18-86
//   jittered mesh (C1/C3) and jump coefficient (C4): SURVEY.md 8(d)
//
// Exported as a plain C ABI (libauxgen.so).
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <stdexcept>
#include <utility>
#include <vector>

namespace {

struct Pt { double x, y; };
struct Trip { int row; int col; double value; };

struct Mesh {
    std::vector<Pt> nodes;
    std::vector<std::array<int, 3>> tris;
    std::vector<int> boundary;
};

struct System {
    Mesh mesh;   // kinds 1-4: the mesh the system was assembled from
    int n = 0;
    std::vector<int> row_ptr, col_idx;
    std::vector<double> values, b, xy;
    // ELL outputs for random_stencil
    std::vector<int> ell_col;
    std::vector<double> ell_val;
};

void csr_from_triplets(System& s, int n, std::vector<Trip>& e) {
    std::sort(e.begin(), e.end(), [](const Trip& a, const Trip& b) {
        return a.row != b.row ? a.row < b.row : a.col < b.col;
    });
    s.n = n;
    s.row_ptr.assign(static_cast<size_t>(n) + 1, 0);
    s.col_idx.clear();
    s.values.clear();
    for (size_t i = 0; i < e.size();) {
        size_t j = i;
        double sum = 0.0;
        while (j < e.size() && e[j].row == e[i].row && e[j].col == e[i].col) sum += e[j++].value;
        s.col_idx.push_back(e[i].col);
        s.values.push_back(sum);
        ++s.row_ptr[e[i].row + 1];
        i = j;
    }
    for (int r = 0; r < n; ++r) s.row_ptr[r + 1] += s.row_ptr[r];
}

Mesh split_mesh(int n) {
    const int w = n + 1;
    const double h = 1.0 / n;
    Mesh m;
    m.nodes.resize(static_cast<size_t>(w) * w);
    for (int j = 0; j < w; ++j)
        for (int i = 0; i < w; ++i) m.nodes[static_cast<size_t>(j) * w + i] = {i * h, j * h};
    m.tris.reserve(static_cast<size_t>(2) * n * n);
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) {
            const int v00 = j * w + i, v10 = v00 + 1, v01 = v00 + w, v11 = v01 + 1;
            m.tris.push_back({v00, v10, v11});
            m.tris.push_back({v00, v11, v01});
        }
    for (int j = 0; j < w; ++j)
        for (int i = 0; i < w; ++i)
            if (i == 0 || j == 0 || i == n || j == n) m.boundary.push_back(j * w + i);
    return m;
}

void detect_boundary(Mesh& m) {
    std::vector<std::pair<int, int>> edges;
    edges.reserve(m.tris.size() * 3);
    for (const auto& t : m.tris)
        for (int v = 0; v < 3; ++v) {
            int a = t[v], b = t[(v + 1) % 3];
            if (a > b) std::swap(a, b);
            edges.emplace_back(a, b);
        }
    std::sort(edges.begin(), edges.end());
    m.boundary.clear();
    for (size_t i = 0; i < edges.size();) {
        size_t j = i;
        while (j < edges.size() && edges[j] == edges[i]) ++j;
        if (j - i == 1) {
            m.boundary.push_back(edges[i].first);
            m.boundary.push_back(edges[i].second);
        }
        i = j;
    }
    std::sort(m.boundary.begin(), m.boundary.end());
    m.boundary.erase(std::unique(m.boundary.begin(), m.boundary.end()), m.boundary.end());
}

Mesh disk_mesh(int n, double cx, double cy, double radius) {
    const Mesh full = split_mesh(n);
    auto inside = [&](const Pt& p) {
        const double dx = p.x - cx, dy = p.y - cy;
        return dx * dx + dy * dy <= radius * radius;
    };
    std::vector<int> remap(full.nodes.size(), -1);
    Mesh d;
    for (const auto& t : full.tris) {
        if (!inside(full.nodes[t[0]]) || !inside(full.nodes[t[1]]) || !inside(full.nodes[t[2]])) continue;
        std::array<int, 3> mp{};
        for (int v = 0; v < 3; ++v) {
            const size_t node = static_cast<size_t>(t[v]);
            if (remap[node] < 0) {
                remap[node] = static_cast<int>(d.nodes.size());
                d.nodes.push_back(full.nodes[node]);
            }
            mp[v] = remap[node];
        }
        d.tris.push_back(mp);
    }
    detect_boundary(d);
    return d;
}

// assemble_fem_triangle with constant source f; jump_kappa > 0 multiplies the
// element stiffness by kappa on the odd cells of an 8x8 checkerboard
// (SURVEY.md 8(d) C4).
void assemble(System& s, const Mesh& m, double f, double jump_kappa) {
    const int n = static_cast<int>(m.nodes.size());
    for (const auto& t : m.tris)
        for (int v : t)
            if (v < 0 || v >= n) throw std::invalid_argument("triangle vertex index out of range");
    std::vector<char> is_b(n, 0);
    for (int v : m.boundary) is_b[v] = 1;
    std::vector<int> interior(n, -1);
    int ni = 0;
    for (int v = 0; v < n; ++v)
        if (!is_b[v]) interior[v] = ni++;
    s.b.assign(ni, 0.0);
    s.xy.resize(static_cast<size_t>(2) * ni);
    for (int v = 0; v < n; ++v)
        if (interior[v] >= 0) {
            s.xy[2 * interior[v]] = m.nodes[v].x;
            s.xy[2 * interior[v] + 1] = m.nodes[v].y;
        }
    std::vector<Trip> e;
    e.reserve(m.tris.size() * 9);
    for (size_t el = 0; el < m.tris.size(); ++el) {
        const auto& t = m.tris[el];
        const Pt p0 = m.nodes[t[0]], p1 = m.nodes[t[1]], p2 = m.nodes[t[2]];
        const double two_area = (p1.x - p0.x) * (p2.y - p0.y) - (p2.x - p0.x) * (p1.y - p0.y);
        const double area = std::abs(two_area) / 2.0;
        if (!(area > 1e-14)) throw std::invalid_argument("degenerate triangle");
        const double gb[3] = {p1.y - p2.y, p2.y - p0.y, p0.y - p1.y};
        const double gc[3] = {p2.x - p1.x, p0.x - p2.x, p1.x - p0.x};
        double kappa = 1.0;
        bool use_k = false;
        if (jump_kappa > 0.0) {
            const double cxx = (p0.x + p1.x + p2.x) / 3.0, cyy = (p0.y + p1.y + p2.y) / 3.0;
            const int bx = std::min(7, static_cast<int>(8.0 * cxx));
            const int by = std::min(7, static_cast<int>(8.0 * cyy));
            if ((bx + by) % 2 == 1) kappa = jump_kappa;
            use_k = true;
        }
        for (int a = 0; a < 3; ++a) {
            const int row = interior[t[a]];
            if (row < 0) continue;
            s.b[row] += f * area / 3.0;
            for (int b = 0; b < 3; ++b) {
                const int col = interior[t[b]];
                if (col < 0) continue;
                const double v = use_k ? (kappa * (gb[a] * gb[b] + gc[a] * gc[b])) / (4.0 * area)
                                       : (gb[a] * gb[b] + gc[a] * gc[b]) / (4.0 * area);
                e.push_back({row, col, v});
            }
        }
    }
    csr_from_triplets(s, ni, e);
}

}  // namespace

extern "C" {

typedef struct auxgen_system auxgen_system;

// kind: 0 = 5-point Poisson gen_poisson_uniform2d(n) (b = h^2)
//       1 = P1 on structured_split_mesh(n)
//       2 = P1 on jittered split mesh (mt19937(seed), U(-amp, amp) * h; C1/C3)
//       3 = P1 on graded_mesh(n, param)               (C2)
//       4 = P1 on disk_mesh(n)                        (inactive cells)
// jump > 0 applies the 8x8 checkerboard coefficient (C4) to kinds 1-4.
auxgen_system* auxgen_make(int kind, int n, double param, unsigned seed, double jump) {
    auto* s = new System;
    try {
        if (kind == 0) {
            const int m = n - 1, N = m * m;
            const double h = 1.0 / n;
            s->xy.resize(static_cast<size_t>(2) * N);
            s->b.resize(N);
            std::vector<Trip> e;
            e.reserve(static_cast<size_t>(5) * N);
            for (int j = 0; j < m; ++j)
                for (int i = 0; i < m; ++i) {
                    const int idx = j * m + i;
                    s->xy[2 * idx] = (i + 1) * h;
                    s->xy[2 * idx + 1] = (j + 1) * h;
                    e.push_back({idx, idx, 4.0});
                    if (i > 0) e.push_back({idx, idx - 1, -1.0});
                    if (i + 1 < m) e.push_back({idx, idx + 1, -1.0});
                    if (j > 0) e.push_back({idx, idx - m, -1.0});
                    if (j + 1 < m) e.push_back({idx, idx + m, -1.0});
                    s->b[idx] = h * h;
                }
            csr_from_triplets(*s, N, e);
            return reinterpret_cast<auxgen_system*>(s);
        }
        Mesh mesh;
        if (kind == 1 || kind == 2 || kind == 3) mesh = split_mesh(n);
        if (kind == 2) {
            std::mt19937 rng(seed);
            std::uniform_real_distribution<double> U(-param, param);
            const double h = 1.0 / n;
            for (int j = 1; j < n; ++j)
                for (int i = 1; i < n; ++i) {
                    Pt& p = mesh.nodes[static_cast<size_t>(j) * (n + 1) + i];
                    p.x += U(rng) * h;
                    p.y += U(rng) * h;
                }
        } else if (kind == 3) {
            for (auto& p : mesh.nodes) {
                p.x = std::pow(p.x, param);
                p.y = std::pow(p.y, param);
            }
        } else if (kind == 4) {
            mesh = disk_mesh(n, 0.5, 0.5, param > 0 ? param : 0.48);
        } else if (kind != 1) {
            throw std::invalid_argument("unknown kind");
        }
        assemble(*s, mesh, 1.0, jump);
        s->mesh = std::move(mesh);
    } catch (...) {
        delete s;
        return nullptr;
    }
    return reinterpret_cast<auxgen_system*>(s);
}

// testgen::random_spd (testgen.hpp:18-35)
auxgen_system* auxgen_random_spd(int n, unsigned seed) {
    auto* s = new System;
    std::mt19937 rng(seed);
    std::uniform_real_distribution<double> unif(-1.0, 1.0);
    const size_t un = static_cast<size_t>(n);
    std::vector<std::vector<double>> m(un, std::vector<double>(un));
    for (auto& row : m)
        for (auto& v : row) v = unif(rng);
    std::vector<Trip> t;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            double v = (i == j) ? static_cast<double>(n) : 0.0;
            for (size_t k = 0; k < un; ++k) v += m[i][k] * m[j][k];
            t.push_back({i, j, v});
        }
    csr_from_triplets(*s, n, t);
    return reinterpret_cast<auxgen_system*>(s);
}

// testgen::random_stencil (testgen.hpp:39-61) with build_stencil_indices
// (hierarchy.hpp:75-91): column-major 9 x 4^k ELL.
auxgen_system* auxgen_random_stencil(int k, unsigned seed) {
    auto* s = new System;
    const int w = 1 << k, n = w * w;
    static const int off[8][2] = {{1, 0}, {1, 1}, {0, 1}, {-1, 1}, {-1, 0}, {-1, -1}, {0, -1}, {1, -1}};
    s->n = n;
    s->ell_col.assign(static_cast<size_t>(9) * n, -1);
    s->ell_val.assign(static_cast<size_t>(9) * n, 0.0);
    for (int i = 0; i < n; ++i) {
        const int t1 = i % w, t2 = i / w;
        s->ell_col[i] = i;
        for (int q = 0; q < 8; ++q) {
            const int u1 = t1 + off[q][0], u2 = t2 + off[q][1];
            if (u1 < 0 || u1 >= w || u2 < 0 || u2 >= w) continue;
            s->ell_col[static_cast<size_t>(q + 1) * n + i] = u2 * w + u1;
        }
    }
    std::mt19937 rng(seed);
    std::uniform_real_distribution<double> unif(0.1, 1.0);
    auto col = [&](int r, int t) { return s->ell_col[static_cast<size_t>(t) * n + r]; };
    auto val = [&](int r, int t) -> double& { return s->ell_val[static_cast<size_t>(t) * n + r]; };
    for (int i = 0; i < n; ++i)
        for (int t = 1; t < 9; ++t) {
            const int j = col(i, t);
            if (j < 0 || j < i) continue;
            const double v = -unif(rng);
            val(i, t) = v;
            for (int q = 1; q < 9; ++q)
                if (col(j, q) == i) val(j, q) = v;
        }
    for (int i = 0; i < n; ++i) {
        double offsum = 0.0;
        for (int t = 1; t < 9; ++t) offsum += std::abs(val(i, t));
        val(i, 0) = offsum + 1.0 + unif(rng);
    }
    return reinterpret_cast<auxgen_system*>(s);
}

// testgen::random_vector (testgen.hpp:79-86)
void auxgen_random_vector(int64_t n, unsigned seed, double lo, double hi, double* out) {
    std::mt19937 rng(seed);
    std::uniform_real_distribution<double> unif(lo, hi);
    for (int64_t i = 0; i < n; ++i) out[i] = unif(rng);
}

int auxgen_n(const auxgen_system* p) { return reinterpret_cast<const System*>(p)->n; }
int64_t auxgen_nnz(const auxgen_system* p) {
    return static_cast<int64_t>(reinterpret_cast<const System*>(p)->values.size());
}
const int* auxgen_row_ptr(const auxgen_system* p) { return reinterpret_cast<const System*>(p)->row_ptr.data(); }
const int* auxgen_col_idx(const auxgen_system* p) { return reinterpret_cast<const System*>(p)->col_idx.data(); }
const double* auxgen_values(const auxgen_system* p) { return reinterpret_cast<const System*>(p)->values.data(); }
const double* auxgen_b(const auxgen_system* p) { return reinterpret_cast<const System*>(p)->b.data(); }
const double* auxgen_xy(const auxgen_system* p) { return reinterpret_cast<const System*>(p)->xy.data(); }
const int* auxgen_ell_col(const auxgen_system* p) { return reinterpret_cast<const System*>(p)->ell_col.data(); }
const double* auxgen_ell_val(const auxgen_system* p) { return reinterpret_cast<const System*>(p)->ell_val.data(); }
// the mesh of kinds 1-4 (node coordinates, triangles, boundary node list)
int auxgen_mesh_nodes(const auxgen_system* p) {
    return static_cast<int>(reinterpret_cast<const System*>(p)->mesh.nodes.size());
}
int auxgen_mesh_tris(const auxgen_system* p) {
    return static_cast<int>(reinterpret_cast<const System*>(p)->mesh.tris.size());
}
int auxgen_mesh_nboundary(const auxgen_system* p) {
    return static_cast<int>(reinterpret_cast<const System*>(p)->mesh.boundary.size());
}
void auxgen_mesh_copy(const auxgen_system* p, double* xy, int* tris, int* boundary) {
    const Mesh& m = reinterpret_cast<const System*>(p)->mesh;
    for (size_t i = 0; i < m.nodes.size(); ++i) {
        xy[2 * i] = m.nodes[i].x;
        xy[2 * i + 1] = m.nodes[i].y;
    }
    for (size_t e = 0; e < m.tris.size(); ++e)
        for (int a = 0; a < 3; ++a) tris[3 * e + a] = m.tris[e][a];
    for (size_t i = 0; i < m.boundary.size(); ++i) boundary[i] = m.boundary[i];
}

void auxgen_free(auxgen_system* p) { delete reinterpret_cast<System*>(p); }

}  // extern "C"

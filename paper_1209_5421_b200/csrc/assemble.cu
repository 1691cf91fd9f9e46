// assemble.cu — device P1 FEM assembly with Dirichlet elimination
// (SURVEY 8(f) rank 1): assemble_fem_triangle (problems.hpp:152-193) and
// csr_from_triplets (sparse.hpp:193-215) on the GPU, the step before setup.
//
//   k_asm_check        vertex / boundary index ranges (argument_error, lowest index)
//   interior numbering exclusive scan of the non-boundary flags (DoFs = interior
//                      nodes in node order, problems.hpp:166-171)
//   k_asm_elements     element geometry (problems.hpp:117-128, same IEEE operations:
//                      the library is built with -fmad=false), degenerate check
//                      (geometry_error, lowest element), 9 stiffness triplets and 3
//                      load contributions per element in the reference's loop order
//   radix sorts        stable LSD sorts by column then row (the triplet order is
//                      (element, a, b), so equal keys keep the reference's emission order)
//   k_asm_segments     duplicates summed sequentially from 0.0 (sparse.hpp:204-206);
//                      the load b[row] += f*area/3 in element order
//
// Bitwise: the sparsity pattern, b, coordinates and every entry summed from one or
// two contributions (all off-diagonal couplings of a conforming mesh).  The reference
// sorts with the unstable std::sort, so the order in which a diagonal's contributions
// are added is an artefact of its introsort; here they are added in element order,
// which can differ from the reference in the last bit (tests/test_gpu_assemble.py).
#include <algorithm>
#include <string>

#include "hier.cuh"
#include "scan_sort.cuh"

struct aux_system {
    int device = 0;
    cudaStream_t stream = nullptr;
    int n = 0;
    long nnz = 0;
    auxb200::DBuf<int> rp, col;
    auxb200::DBuf<double> val, b, xy;
    ~aux_system() {
        if (stream) cudaStreamSynchronize(stream);
        rp.release();
        col.release();
        val.release();
        b.release();
        xy.release();
        if (stream) cudaStreamDestroy(stream);
    }
};

namespace auxb200 {

namespace {

constexpr int kT = 256;
inline unsigned grid_for(long n) {
    long b = (n + kT - 1) / kT;
    if (b < 1) b = 1;
    if (b > 148L * 64) b = 148L * 64;
    return static_cast<unsigned>(b);
}
#define GSTRIDE(i, n) for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < (n); i += (long)gridDim.x * blockDim.x)

template <class T>
T read1(const T* d, cudaStream_t s) {
    T v;
    AUX_CUDA(cudaMemcpyAsync(&v, d, sizeof(T), cudaMemcpyDeviceToHost, s));
    AUX_CUDA(cudaStreamSynchronize(s));
    return v;
}

__global__ void k_asm_check(const int* __restrict__ tris, long ne, const int* __restrict__ bnd, int nb, int n,
                            unsigned long long* err, int* __restrict__ is_b) {
    GSTRIDE(e, ne) {
        for (int a = 0; a < 3; ++a) {
            const int v = tris[3 * e + a];
            if (v < 0 || v >= n) atomicMin(err, (unsigned long long)e);
        }
    }
    GSTRIDE(i, nb) {
        const int v = bnd[i];
        if (v < 0 || v >= n) atomicMin(err + 1, (unsigned long long)i);
        else is_b[v] = 1;
    }
}

__global__ void k_asm_interior(const int* __restrict__ is_b, int n, int* __restrict__ flag) {
    GSTRIDE(v, n) flag[v] = is_b[v] ? 0 : 1;
}

__global__ void k_asm_number(const int* __restrict__ flag, const int* __restrict__ pos, int n,
                             const double* __restrict__ nodes, int* __restrict__ interior, double* __restrict__ xy) {
    GSTRIDE(v, n) {
        if (flag[v]) {
            const int i = pos[v];
            interior[v] = i;
            xy[2 * (long)i] = nodes[2 * v];
            xy[2 * (long)i + 1] = nodes[2 * v + 1];
        } else {
            interior[v] = -1;
        }
    }
}

// one element: geometry (problems.hpp:117-128), 9 stiffness triplets (row, col,
// value) in (a, b) order and 3 load contributions; entries touching a boundary
// node get the key `ni` (sorted past every real key and dropped)
__global__ void k_asm_elements(const int* __restrict__ tris, long ne, const double* __restrict__ nodes,
                               const int* __restrict__ interior, int ni, double f, double jump,
                               unsigned* __restrict__ krow, unsigned* __restrict__ kcol, double* __restrict__ kval,
                               unsigned* __restrict__ brow, double* __restrict__ bval,
                               unsigned long long* degenerate) {
    GSTRIDE(e, ne) {
        const int t0 = tris[3 * e], t1 = tris[3 * e + 1], t2 = tris[3 * e + 2];
        const double p0x = nodes[2 * t0], p0y = nodes[2 * t0 + 1];
        const double p1x = nodes[2 * t1], p1y = nodes[2 * t1 + 1];
        const double p2x = nodes[2 * t2], p2y = nodes[2 * t2 + 1];
        const double two_area = (p1x - p0x) * (p2y - p0y) - (p2x - p0x) * (p1y - p0y);
        const double area = fabs(two_area) / 2.0;
        if (!(area > 1e-14)) atomicMin(degenerate, (unsigned long long)e);
        const double gb[3] = {p1y - p2y, p2y - p0y, p0y - p1y};
        const double gc[3] = {p2x - p1x, p0x - p2x, p1x - p0x};
        double kappa = 1.0;
        const bool use_k = jump > 0.0;   // harness C4 checkerboard (problems.cpp)
        if (use_k) {
            const double cx = (p0x + p1x + p2x) / 3.0, cy = (p0y + p1y + p2y) / 3.0;
            const int bx = min(7, (int)(8.0 * cx)), by = min(7, (int)(8.0 * cy));
            if ((bx + by) % 2 == 1) kappa = jump;
        }
        const int vv[3] = {t0, t1, t2};
        for (int a = 0; a < 3; ++a) {
            const int row = interior[vv[a]];
            brow[3 * e + a] = row < 0 ? (unsigned)ni : (unsigned)row;
            bval[3 * e + a] = f * area / 3.0;
            for (int b = 0; b < 3; ++b) {
                const int col = interior[vv[b]];
                const long k = 9 * e + 3 * a + b;
                const bool keep = row >= 0 && col >= 0;
                krow[k] = keep ? (unsigned)row : (unsigned)ni;
                kcol[k] = keep ? (unsigned)col : (unsigned)ni;
                kval[k] = use_k ? (kappa * (gb[a] * gb[b] + gc[a] * gc[b])) / (4.0 * area)
                                : (gb[a] * gb[b] + gc[a] * gc[b]) / (4.0 * area);
            }
        }
    }
}

__global__ void k_gather_u(const unsigned* __restrict__ src, const int* __restrict__ idx, long n,
                           unsigned* __restrict__ dst) {
    GSTRIDE(i, n) dst[i] = src[idx[i]];
}

// first entry of each (row, col) run among the real keys
__global__ void k_asm_heads(const unsigned* __restrict__ krow, const unsigned* __restrict__ kcol,
                            const int* __restrict__ idx, long m, unsigned ni, int* __restrict__ head) {
    GSTRIDE(i, m) {
        const int k = idx[i];
        const unsigned r = krow[k], c = kcol[k];
        bool h = r < ni;
        if (h && i > 0) {
            const int kp = idx[i - 1];
            h = !(krow[kp] == r && kcol[kp] == c);
        }
        head[i] = h ? 1 : 0;
    }
}

// sum each run sequentially from 0.0 (sparse.hpp:204-206), emit column and row count
__global__ void k_asm_segments(const unsigned* __restrict__ krow, const unsigned* __restrict__ kcol,
                               const double* __restrict__ kval, const int* __restrict__ idx,
                               const int* __restrict__ head, const int* __restrict__ hpos, long m,
                               int* __restrict__ col, double* __restrict__ val, int* __restrict__ rowcnt) {
    GSTRIDE(i, m) {
        if (!head[i]) continue;
        const int k = idx[i];
        const unsigned r = krow[k], c = kcol[k];
        double sum = 0.0;
        for (long j = i; j < m; ++j) {
            const int kj = idx[j];
            if (krow[kj] != r || kcol[kj] != c) break;
            sum += kval[kj];
        }
        const int o = hpos[i];
        col[o] = (int)c;
        val[o] = sum;
        atomicAdd(&rowcnt[r], 1);
    }
}

// b[row] = sum of f*area/3 over the elements of the node, in element order
__global__ void k_asm_load(const unsigned* __restrict__ brow, const double* __restrict__ bval,
                           const int* __restrict__ idx, long m, unsigned ni, double* __restrict__ b) {
    GSTRIDE(i, m) {
        const int k = idx[i];
        const unsigned r = brow[k];
        if (r >= ni) continue;
        if (i > 0 && brow[idx[i - 1]] == r) continue;
        double sum = 0.0;
        for (long j = i; j < m; ++j) {
            const int kj = idx[j];
            if (brow[kj] != r) break;
            sum += bval[kj];
        }
        b[r] = sum;
    }
}

// ---- galerkin_dense (hierarchy.hpp:239-247): one key
// agg(i) * n_agg + agg(j) per stored entry, emitted in storage order (rows
// ascending, entries in row order), a stable radix sort, then every run summed
// sequentially from 0.0 -- the reference's accumulation order per element.
__global__ void k_gd_keys(const int* __restrict__ rp, const int* __restrict__ col, const int* __restrict__ agg,
                          int n, int n_agg, unsigned* __restrict__ key, unsigned long long* bad) {
    GSTRIDE(i, n) {
        const int ai = agg[i];
        if (ai < 0 || ai >= n_agg) atomicMin(bad, (unsigned long long)i);
        for (int p = rp[i]; p < rp[i + 1]; ++p) {
            const int aj = agg[col[p]];
            key[p] = (unsigned)ai * (unsigned)n_agg + (unsigned)aj;
        }
    }
}
__global__ void k_gd_sum(const unsigned* __restrict__ skey, const int* __restrict__ idx,
                         const double* __restrict__ v, long m, double* __restrict__ C) {
    GSTRIDE(i, m) {
        if (i > 0 && skey[i - 1] == skey[i]) continue;
        double sum = 0.0;
        for (long j = i; j < m && skey[j] == skey[i]; ++j) sum += v[idx[j]];
        C[skey[i]] = sum;
    }
}

int bits_for(unsigned long v) {
    int b = 1;
    while ((1ul << b) <= v) ++b;
    return b;
}

void assemble(aux_system* S, const double* nodes_d, int n, const int* tris_d, long ne, const int* bnd_d, int nb,
              double f, double jump) {
    cudaStream_t s = S->stream;
    DBuf<unsigned long long> err(3);
    AUX_CUDA(cudaMemsetAsync(err.p, 0xff, 3 * sizeof(unsigned long long), s));
    DBuf<int> is_b(std::max(n, 1));
    AUX_CUDA(cudaMemsetAsync(is_b.p, 0, sizeof(int) * std::max(n, 1), s));
    k_asm_check<<<grid_for(std::max<long>(ne, nb)), kT, 0, s>>>(tris_d, ne, bnd_d, nb, n, err.p, is_b.p);
    AUX_LAUNCHED(1);
    unsigned long long e[2];
    AUX_CUDA(cudaMemcpyAsync(e, err.p, sizeof e, cudaMemcpyDeviceToHost, s));
    AUX_CUDA(cudaStreamSynchronize(s));
    if (e[0] != ~0ull) throw_aux(AUX_ARGUMENT_ERROR, "triangle vertex index out of range");
    if (e[1] != ~0ull) throw_aux(AUX_ARGUMENT_ERROR, "boundary node index out of range");
    // interior numbering and coordinates
    DBuf<int> flag(std::max(n, 1)), pos(n + 1), interior(std::max(n, 1));
    k_asm_interior<<<grid_for(n), kT, 0, s>>>(is_b.p, n, flag.p);
    AUX_LAUNCHED(1);
    exclusive_scan(flag.p, pos.p, n, s);
    const int ni = read1(pos.p + n, s);
    S->n = ni;
    S->xy.alloc(2 * (size_t)std::max(ni, 1));
    S->b.alloc(std::max(ni, 1));
    AUX_CUDA(cudaMemsetAsync(S->b.p, 0, sizeof(double) * std::max(ni, 1), s));
    k_asm_number<<<grid_for(n), kT, 0, s>>>(flag.p, pos.p, n, nodes_d, interior.p, S->xy.p);
    AUX_LAUNCHED(1);
    // element triplets
    const long m = 9 * ne, mb = 3 * ne;
    DBuf<unsigned> krow(std::max<long>(m, 1)), kcol(std::max<long>(m, 1)), brow(std::max<long>(mb, 1));
    DBuf<double> kval(std::max<long>(m, 1)), bval(std::max<long>(mb, 1));
    if (ne > 0) {
        k_asm_elements<<<grid_for(ne), kT, 0, s>>>(tris_d, ne, nodes_d, interior.p, ni, f, jump, krow.p, kcol.p,
                                                   kval.p, brow.p, bval.p, err.p + 2);
        AUX_LAUNCHED(1);
    }
    const unsigned long long deg = read1(err.p + 2, s);
    if (deg != ~0ull) throw_aux(AUX_GEOMETRY_ERROR, "triangle " + std::to_string(deg) + " is degenerate");
    const int nbits = bits_for((unsigned long)ni);
    // stable (row, col) order: sort by column, then stably by row
    DBuf<int> idx(std::max<long>(m, 1));
    DBuf<unsigned> key(std::max<long>(m, 1));
    AUX_CUDA(cudaMemcpyAsync(key.p, kcol.p, sizeof(unsigned) * m, cudaMemcpyDeviceToDevice, s));
    radix_sort_pairs(key.p, idx.p, m, nbits, s, true);
    k_gather_u<<<grid_for(m), kT, 0, s>>>(krow.p, idx.p, m, key.p);
    AUX_LAUNCHED(1);
    radix_sort_pairs(key.p, idx.p, m, nbits, s, false);
    DBuf<int> head(std::max<long>(m, 1)), hpos(m + 1);
    k_asm_heads<<<grid_for(m), kT, 0, s>>>(krow.p, kcol.p, idx.p, m, (unsigned)ni, head.p);
    AUX_LAUNCHED(1);
    exclusive_scan(head.p, hpos.p, m, s);
    S->nnz = read1(hpos.p + m, s);
    S->col.alloc(std::max<long>(S->nnz, 1));
    S->val.alloc(std::max<long>(S->nnz, 1));
    DBuf<int> cnt(std::max(ni, 1));
    AUX_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int) * std::max(ni, 1), s));
    k_asm_segments<<<grid_for(m), kT, 0, s>>>(krow.p, kcol.p, kval.p, idx.p, head.p, hpos.p, m, S->col.p, S->val.p,
                                              cnt.p);
    AUX_LAUNCHED(1);
    S->rp.alloc(ni + 1);
    exclusive_scan(cnt.p, S->rp.p, ni, s);
    // load vector, element order per row
    DBuf<int> bidx(std::max<long>(mb, 1));
    DBuf<unsigned> bkey(std::max<long>(mb, 1));
    AUX_CUDA(cudaMemcpyAsync(bkey.p, brow.p, sizeof(unsigned) * mb, cudaMemcpyDeviceToDevice, s));
    radix_sort_pairs(bkey.p, bidx.p, mb, nbits, s, true);
    k_asm_load<<<grid_for(mb), kT, 0, s>>>(brow.p, bval.p, bidx.p, mb, (unsigned)ni, S->b.p);
    AUX_LAUNCHED(1);
    AUX_CUDA(cudaStreamSynchronize(s));
}

}  // namespace

}  // namespace auxb200

using namespace auxb200;

extern "C" {

aux_status aux_assemble_p1(const double* nodes_xy, int32_t n_nodes, const int32_t* tris, int64_t n_tris,
                           const int32_t* boundary, int32_t n_boundary, double f, double jump, int32_t device,
                           aux_system** out, char* msg, size_t msg_len) {
    *out = nullptr;
    aux_system* S = nullptr;
    try {
        if (n_nodes < 0 || n_tris < 0 || n_boundary < 0) throw_aux(AUX_SIZE_ERROR, "assemble: negative size");
        S = new aux_system();
        S->device = device;
        AUX_CUDA(cudaSetDevice(device));
        AUX_CUDA(cudaStreamCreateWithFlags(&S->stream, cudaStreamNonBlocking));
        DBuf<double> nd(2 * (size_t)std::max(n_nodes, 1));
        DBuf<int> td(3 * (size_t)std::max<int64_t>(n_tris, 1)), bd(std::max(n_boundary, 1));
        if (n_nodes)
            AUX_CUDA(cudaMemcpyAsync(nd.p, nodes_xy, sizeof(double) * 2 * n_nodes, cudaMemcpyHostToDevice, S->stream));
        if (n_tris)
            AUX_CUDA(cudaMemcpyAsync(td.p, tris, sizeof(int) * 3 * n_tris, cudaMemcpyHostToDevice, S->stream));
        if (n_boundary)
            AUX_CUDA(cudaMemcpyAsync(bd.p, boundary, sizeof(int) * n_boundary, cudaMemcpyHostToDevice, S->stream));
        assemble(S, nd.p, n_nodes, td.p, n_tris, bd.p, n_boundary, f, jump);
        *out = S;
        if (msg && msg_len) msg[0] = 0;
        return AUX_OK;
    } catch (const AuxError& e) {
        delete S;
        if (msg && msg_len) std::snprintf(msg, msg_len, "%s", e.what());
        return e.code;
    } catch (const std::exception& e) {
        delete S;
        if (msg && msg_len) std::snprintf(msg, msg_len, "%s", e.what());
        return AUX_INTERNAL_ERROR;
    }
}

aux_status aux_system_info(const aux_system* S, int32_t* n, int64_t* nnz) {
    *n = S->n;
    *nnz = S->nnz;
    return AUX_OK;
}

aux_status aux_system_device(const aux_system* S, aux_csr_view* A, const double** b, const double** xy) {
    A->n_rows = A->n_cols = S->n;
    A->nnz = S->nnz;
    A->row_ptr = S->rp.p;
    A->col_idx = S->col.p;
    A->values = S->val.p;
    *b = S->b.p;
    *xy = S->xy.p;
    return AUX_OK;
}

aux_status aux_system_copy(const aux_system* S, int32_t* row_ptr, int32_t* col_idx, double* values, double* b,
                           double* xy) {
    try {
        AUX_CUDA(cudaMemcpy(row_ptr, S->rp.p, sizeof(int) * (S->n + 1), cudaMemcpyDeviceToHost));
        if (S->nnz) {
            AUX_CUDA(cudaMemcpy(col_idx, S->col.p, sizeof(int) * S->nnz, cudaMemcpyDeviceToHost));
            AUX_CUDA(cudaMemcpy(values, S->val.p, sizeof(double) * S->nnz, cudaMemcpyDeviceToHost));
        }
        if (S->n) {
            AUX_CUDA(cudaMemcpy(b, S->b.p, sizeof(double) * S->n, cudaMemcpyDeviceToHost));
            AUX_CUDA(cudaMemcpy(xy, S->xy.p, sizeof(double) * 2 * S->n, cudaMemcpyDeviceToHost));
        }
        return AUX_OK;
    } catch (const AuxError& e) {
        return e.code;
    }
}

void aux_system_destroy(aux_system* S) { delete S; }

aux_status aux_galerkin_dense(const aux_csr_view* A, const int32_t* agg_of, int64_t n_agg_of, int32_t n_agg,
                              int32_t device, double* C, char* msg, size_t msg_len) {
    cudaStream_t s = nullptr;
    try {
        if (n_agg_of != A->n_rows) throw_aux(AUX_SIZE_ERROR, "galerkin_dense: map does not match matrix");
        if (n_agg < 1 || (long)n_agg * n_agg >= (1l << 32))
            throw_aux(AUX_CAPACITY_ERROR, "galerkin_dense: aggregate count out of range for a dense result");
        AUX_CUDA(cudaSetDevice(device));
        AUX_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        const int n = A->n_rows;
        const long m = A->nnz;
        DBuf<int> rp(n + 1), col(std::max<long>(m, 1)), agg(std::max(n, 1)), idx(std::max<long>(m, 1));
        DBuf<double> v(std::max<long>(m, 1)), Cd((size_t)n_agg * n_agg);
        DBuf<unsigned> key(std::max<long>(m, 1));
        DBuf<unsigned long long> bad(1);
        AUX_CUDA(cudaMemcpyAsync(rp.p, A->row_ptr, sizeof(int) * (n + 1), cudaMemcpyHostToDevice, s));
        if (m) {
            AUX_CUDA(cudaMemcpyAsync(col.p, A->col_idx, sizeof(int) * m, cudaMemcpyHostToDevice, s));
            AUX_CUDA(cudaMemcpyAsync(v.p, A->values, sizeof(double) * m, cudaMemcpyHostToDevice, s));
        }
        if (n) AUX_CUDA(cudaMemcpyAsync(agg.p, agg_of, sizeof(int) * n, cudaMemcpyHostToDevice, s));
        AUX_CUDA(cudaMemsetAsync(Cd.p, 0, sizeof(double) * (size_t)n_agg * n_agg, s));
        AUX_CUDA(cudaMemsetAsync(bad.p, 0xff, sizeof(unsigned long long), s));
        k_gd_keys<<<grid_for(n), kT, 0, s>>>(rp.p, col.p, agg.p, n, n_agg, key.p, bad.p);
        AUX_LAUNCHED(1);
        if (read1(bad.p, s) != ~0ull) throw_aux(AUX_ARGUMENT_ERROR, "galerkin_dense: aggregate id out of range");
        if (m) {
            radix_sort_pairs(key.p, idx.p, m, bits_for((unsigned long)n_agg * n_agg), s, true);
            k_gd_sum<<<grid_for(m), kT, 0, s>>>(key.p, idx.p, v.p, m, Cd.p);
            AUX_LAUNCHED(1);
        }
        AUX_CUDA(cudaMemcpyAsync(C, Cd.p, sizeof(double) * (size_t)n_agg * n_agg, cudaMemcpyDeviceToHost, s));
        AUX_CUDA(cudaStreamSynchronize(s));
        cudaStreamDestroy(s);
        if (msg && msg_len) msg[0] = 0;
        return AUX_OK;
    } catch (const AuxError& e) {
        if (s) { cudaStreamSynchronize(s); cudaStreamDestroy(s); }
        if (msg && msg_len) std::snprintf(msg, msg_len, "%s", e.what());
        return e.code;
    }
}

}  // extern "C"

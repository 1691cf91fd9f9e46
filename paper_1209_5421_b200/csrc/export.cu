// export.cu — read access to the device hierarchy in the reference's layout
// and indexing (Level / AggregationMap / EllMatrix / ColorSchedule /
// BlockFactors / LuFactors, hierarchy.hpp:288-309).  Used by the parity tests
// and by callers that inspect Hierarchy internals (test_hierarchy.cpp:255-301).
// Index conversion runs on the host over downloaded arrays; the block factors
// are recomputed on the device with the reference's loop (lu_factor order).
#include <cstring>
#include <vector>

#include "lu.cuh"
#include "setup.cuh"

namespace auxb200 {

namespace {

template <class T>
std::vector<T> down(const T* d, size_t n, cudaStream_t s) {
    std::vector<T> v(n);
    if (n) {
        AUX_CUDA(cudaMemcpyAsync(v.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost, s));
        AUX_CUDA(cudaStreamSynchronize(s));
    }
    return v;
}

// factor_blocks (smoother.hpp:129-156) for every aggregate, lexicographic order.
__global__ void k_export_blocks(int nL, Geo g, const int* __restrict__ bptr, const int* __restrict__ rp,
                                const int* __restrict__ col, const double* __restrict__ v,
                                const long long* __restrict__ off, const int* __restrict__ mptr,
                                double* __restrict__ lu, int* __restrict__ perm) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nL; r += gridDim.x * blockDim.x) {
        const int gcm = cm_of_lex(g, r);
        const int r0 = bptr[gcm], s = bptr[gcm + 1] - r0;
        if (s == 0) continue;
        double* a = lu + off[r];
        for (long e = 0; e < (long)s * s; ++e) a[e] = 0.0;
        for (int q = 0; q < s; ++q)
            for (int p = rp[r0 + q]; p < rp[r0 + q + 1]; ++p) {
                const unsigned c = (unsigned)(col[p] - r0);
                if (c < (unsigned)s) a[(size_t)q * s + c] = v[p];
            }
        seq_lu_factor(a, perm + mptr[r], s);
    }
}

}  // namespace

void level_info(const aux_hierarchy* h, int l, aux_level_info* o) {
    std::memset(o, 0, sizeof *o);
    const Level& L = h->lv[l];
    o->n = L.n;
    o->nnz = L.nnz;
    o->structured = L.structured ? 1 : 0;
    const bool last = l == (int)h->lv.size() - 1;
    if (l == 0) {
        o->k = h->direct_only ? 0 : h->depth + 1;
        if (!h->direct_only) {
            o->has_map = 1;
            o->map_level = h->depth;
            o->n_aggregates = 1 << (2 * h->depth);
            o->n_items = o->n_aggregates;
            const std::vector<int> bp = down(h->fine.bptr.p, (size_t)o->n_aggregates + 1, h->stream);
            long pool = 0;
            for (int g = 0; g < o->n_aggregates; ++g) {
                const long s = bp[g + 1] - bp[g];
                pool += s * s;
            }
            o->block_pool = pool;
        }
    } else {
        o->k = L.k;
        o->n_items = L.n;
        if (!last) {
            o->has_map = 1;
            o->map_level = L.k;
            o->n_aggregates = 1 << (2 * (L.k - 1));
        }
    }
}

void export_level(const aux_hierarchy* h, int l, aux_level_export* x) {
    cudaStream_t s = h->stream;
    aux_level_info info;
    level_info(h, l, &info);
    const int n = info.n;
    if (l == 0) {
        if (x->active) std::memset(x->active, 1, (size_t)n);
        if (h->direct_only) return;
        const Finest& F = h->fine;
        const Geo gL = h->lv[1].geo;
        const int nL = gL.n;
        const std::vector<int> bp = down(F.bptr.p, (size_t)nL + 1, s);
        const std::vector<int> perm = down(F.perm.p, (size_t)n, s);
        const std::vector<int> lexrow = down(F.lex_of_row.p, (size_t)n, s);
        std::vector<int> mptr(nL + 1, 0);
        std::vector<long long> off(nL + 1, 0);
        for (int r = 0; r < nL; ++r) {
            const int g = cm_of_lex(gL, r);
            const int sz = bp[g + 1] - bp[g];
            mptr[r + 1] = mptr[r] + sz;
            off[r + 1] = off[r] + (long long)sz * sz;
        }
        if (x->agg_of)
            for (int i = 0; i < n; ++i) x->agg_of[perm[i]] = lexrow[i];
        if (x->member_ptr) std::memcpy(x->member_ptr, mptr.data(), sizeof(int) * (nL + 1));
        if (x->member_idx)
            for (int r = 0; r < nL; ++r) {
                const int g = cm_of_lex(gL, r);
                for (int q = bp[g]; q < bp[g + 1]; ++q) x->member_idx[mptr[r] + (q - bp[g])] = perm[q];
            }
        if (x->item_color)
            for (int r = 0; r < nL; ++r) {
                const int g = cm_of_lex(gL, r);
                x->item_color[r] = bp[g + 1] > bp[g] ? (g >> gL.lq) : -1;
            }
        if (x->block_size)
            for (int r = 0; r < nL; ++r) x->block_size[r] = mptr[r + 1] - mptr[r];
        if (x->block_offset) std::memcpy(x->block_offset, off.data(), sizeof(long long) * (nL + 1));
        if (x->block_lu || x->block_perm) {
            DBuf<long long> doff(nL + 1);
            DBuf<int> dmptr(nL + 1);
            DBuf<double> dlu(std::max<long long>(off[nL], 1));
            DBuf<int> dperm(std::max(n, 1));
            AUX_CUDA(cudaMemcpyAsync(doff.p, off.data(), sizeof(long long) * (nL + 1), cudaMemcpyHostToDevice, s));
            AUX_CUDA(cudaMemcpyAsync(dmptr.p, mptr.data(), sizeof(int) * (nL + 1), cudaMemcpyHostToDevice, s));
            k_export_blocks<<<(nL + 127) / 128, 128, 0, s>>>(nL, gL, F.bptr.p, F.rp.p, F.col.p, F.v.p, doff.p, dmptr.p,
                                                             dlu.p, dperm.p);
            AUX_LAUNCHED(1);
            AUX_CUDA(cudaGetLastError());
            if (x->block_lu && off[nL] > 0)
                AUX_CUDA(cudaMemcpyAsync(x->block_lu, dlu.p, sizeof(double) * off[nL], cudaMemcpyDeviceToHost, s));
            if (x->block_perm)
                AUX_CUDA(cudaMemcpyAsync(x->block_perm, dperm.p, sizeof(int) * n, cudaMemcpyDeviceToHost, s));
            AUX_CUDA(cudaStreamSynchronize(s));
        }
        return;
    }
    const Level& L = h->lv[l];
    const Geo g = L.geo;
    const int w = 1 << g.k;
    const std::vector<uint8_t> act = down(L.active.p, (size_t)n, s);
    auto cm = [&](int lex) { return cm_of_lex(g, lex); };
    if (x->active)
        for (int r = 0; r < n; ++r) x->active[r] = act[cm(r)];
    if (x->item_color)
        for (int r = 0; r < n; ++r) x->item_color[r] = act[cm(r)] ? ((r % w) % 2 + 2 * ((r / w) % 2)) : -1;
    if (x->ell_col)
        for (int r = 0; r < n; ++r) {
            const int t1 = r % w, t2 = r / w;
            x->ell_col[r] = r;
            for (int t = 1; t < 9; ++t) {
                const int u1 = t1 + stencil_dx(t), u2 = t2 + stencil_dy(t);
                const bool in = act[cm(r)] && u1 >= 0 && u1 < w && u2 >= 0 && u2 < w;
                x->ell_col[(size_t)t * n + r] = in ? u2 * w + u1 : -1;
            }
        }
    if (x->ell_val) {
        const std::vector<double> v = down(L.val.p, (size_t)9 * n, s);
        for (int r = 0; r < n; ++r)
            for (int t = 0; t < 9; ++t) x->ell_val[(size_t)t * n + r] = v[(size_t)t * n + cm(r)];
    }
    if (info.has_map) {
        const int wc = w / 2;
        if (x->agg_of)
            for (int r = 0; r < n; ++r) x->agg_of[r] = ((r / w) / 2) * wc + (r % w) / 2;
        if (x->member_ptr)
            for (int i = 0; i <= info.n_aggregates; ++i) x->member_ptr[i] = 4 * i;
        if (x->member_idx)
            for (int i = 0; i < info.n_aggregates; ++i) {
                const int T1 = i % wc, T2 = i / wc;
                x->member_idx[4 * i + 0] = (2 * T2) * w + 2 * T1;
                x->member_idx[4 * i + 1] = (2 * T2) * w + 2 * T1 + 1;
                x->member_idx[4 * i + 2] = (2 * T2 + 1) * w + 2 * T1;
                x->member_idx[4 * i + 3] = (2 * T2 + 1) * w + 2 * T1 + 1;
            }
    }
}

void export_coarsest(const aux_hierarchy* h, int* n, double* lu, int* perm) {
    *n = h->nc;
    if (lu) {
        AUX_CUDA(cudaMemcpyAsync(lu, h->c_lu.p, sizeof(double) * h->nc * h->nc, cudaMemcpyDeviceToHost, h->stream));
    }
    if (perm) AUX_CUDA(cudaMemcpyAsync(perm, h->c_perm.p, sizeof(int) * h->nc, cudaMemcpyDeviceToHost, h->stream));
    AUX_CUDA(cudaStreamSynchronize(h->stream));
}

}  // namespace auxb200

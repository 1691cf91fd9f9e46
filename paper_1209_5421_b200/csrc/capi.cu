// capi.cu — the C ABI (include/auxamg_b200.h).  Every entry point converts
// the library's AuxError into the status code of the matching reference
// exception class (errors.hpp:13-76) plus its message.
#include <chrono>
#include <cstring>
#include <new>
#include <string>

#include "comm.cuh"
#include "setup.cuh"

namespace auxb200 {
std::atomic<int64_t> g_launches{0};
}

using namespace auxb200;

namespace {

aux_status fill(char* msg, size_t len, aux_status st, const char* what) {
    if (msg && len) std::snprintf(msg, len, "%s", what);
    return st;
}

template <class F>
aux_status guarded(char* msg, size_t len, F&& f) {
    try {
        f();
        if (msg && len) msg[0] = 0;
        return AUX_OK;
    } catch (const AuxError& e) {
        return fill(msg, len, e.code, e.what());
    } catch (const std::bad_alloc& e) {
        return fill(msg, len, AUX_INTERNAL_ERROR, "host allocation failed");
    } catch (const std::exception& e) {
        return fill(msg, len, AUX_INTERNAL_ERROR, e.what());
    }
}

aux_hierarchy* make_h(const aux_setup_opts* o, const aux_gpu_opts* g) {
    if (g && (g->block_solve < 0 || g->block_solve > 1 || g->coarse_solve < 0 || g->coarse_solve > 1))
        throw_aux(AUX_ARGUMENT_ERROR, "aux_gpu_opts: block_solve and coarse_solve must be 0 or 1");
    auto* h = new aux_hierarchy();
    aux_default_setup_opts(&h->opts);
    aux_default_gpu_opts(&h->gpu);
    if (o) h->opts = *o;
    if (g) h->gpu = *g;
    AUX_CUDA(cudaSetDevice(h->gpu.device));
    AUX_CUDA(cudaDeviceGetAttribute(&h->sm_count, cudaDevAttrMultiProcessorCount, h->gpu.device));
    {
        HostCallTimer tm("stream_pool_get");
        h->stream = stream_pool_get();
    }
    h->red_partials.alloc((size_t)kMaxRedBlocks * 4);
    h->red_ticket.alloc(1);
    AUX_CUDA(cudaMemsetAsync(h->red_ticket.p, 0, sizeof(unsigned int), h->stream));
    return h;
}

}  // namespace

aux_hierarchy::~aux_hierarchy() {
    HostCallTimer tm_all("destroy (total)");
    if (stream) cudaStreamSynchronize(stream);   // no launch of the graph still in flight
    if (graph) {
        HostCallTimer tm("graph_exec_release");
        graph_exec_release(graph);
    }
    for (int k = 0; k < kProfKinds; ++k) {
        for (auto e : prof.ev_begin[k]) cudaEventDestroy(e);
        for (auto e : prof.ev_end[k]) cudaEventDestroy(e);
    }
    if (stream) cudaStreamSynchronize(stream);
    if (dist.owns_comm) delete dist.comm;
    dist.comm = nullptr;
    // DBufs free themselves; the stream goes last
    fine = Finest();
    lv.clear();
    w_p.clear();
    w_ap.clear();
    if (stream) {
        HostCallTimer tm("stream_pool_put");
        stream_pool_put(stream);   // synchronised above
    }
}

extern "C" {

void aux_default_setup_opts(aux_setup_opts* o) {
    o->coarsest_size = 64;
    o->strict_locality = 0;
    o->lump_locality = 0;
    o->symmetry_tol = 1e-10;
}

void aux_default_cycle_opts(aux_cycle_opts* o) {
    o->n_inner = 2;
    o->pre_sweeps = 1;
    o->post_sweeps = 1;
    o->max_outer = 100;
    o->rtol = 1e-6;
    o->max_directions = 0;
}

void aux_default_gpu_opts(aux_gpu_opts* o) {
    std::memset(o, 0, sizeof *o);
    o->device = 0;
    o->coarse_solve = 0;
    o->fused_max_cells = -1;
    o->use_graphs = 1;
    o->block_solve = 0;
    o->tile_kernels = 1;
    o->cluster_tier = 1;
}

const char* aux_version(void) { return "auxamg_b200 0.1 (sm_100a)"; }

void aux_set_num_threads(int32_t) {}

aux_status aux_setup_device(const aux_csr_view* A, const double* xy, int64_t n_points, const aux_setup_opts* opts,
                            const aux_gpu_opts* gpu, aux_hierarchy** out, char* msg, size_t msg_len) {
    *out = nullptr;
    aux_hierarchy* h = nullptr;
    const aux_status st = guarded(msg, msg_len, [&] {
        DeviceGuard dg(gpu ? gpu->device : 0);
        h = make_h(opts, gpu);
        const auto t0 = std::chrono::steady_clock::now();
        setup_device(h, A, xy, (long)n_points);
        h->last_setup_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    });
    if (st != AUX_OK) {
        delete h;
        return st;
    }
    *out = h;
    return AUX_OK;
}

aux_status aux_setup(const aux_csr_view* A, const double* xy, int64_t n_points, const aux_setup_opts* opts,
                     const aux_gpu_opts* gpu, aux_hierarchy** out, char* msg, size_t msg_len) {
    *out = nullptr;
    aux_hierarchy* h = nullptr;
    const aux_status st = guarded(msg, msg_len, [&] {
        DeviceGuard dg(gpu ? gpu->device : 0);
        h = make_h(opts, gpu);
        const auto t0 = std::chrono::steady_clock::now();
        if (A->n_rows < 0 || A->nnz < 0) throw_aux(AUX_SIZE_ERROR, "setup_hierarchy: negative size");
        const long n = A->n_rows;
        DBuf<int> rp(n + 1), col(A->nnz);
        DBuf<double> v(A->nnz), xy_d(2 * std::max<long>(n_points, 0));
        // structure and coordinates first on the setup stream; the values (half
        // the bytes) on a second stream, so the structure check and the
        // coordinate-only phase of setup overlap their copy
        struct Side {
            cudaStream_t s = nullptr;
            cudaEvent_t e = nullptr;
            ~Side() {   // (destroyed before v: an error thrown mid-copy still waits for it)
                if (s) cudaStreamSynchronize(s);
                if (e) cudaEventDestroy(e);
                if (s) stream_pool_put(s);
            }
        } side;
        side.s = stream_pool_get();
        AUX_CUDA(cudaEventCreateWithFlags(&side.e, cudaEventDisableTiming));
        AUX_CUDA(cudaMemcpyAsync(rp.p, A->row_ptr, sizeof(int) * (n + 1), cudaMemcpyHostToDevice, h->stream));
        if (n_points > 0)
            AUX_CUDA(cudaMemcpyAsync(xy_d.p, xy, sizeof(double) * 2 * n_points, cudaMemcpyHostToDevice, h->stream));
        if (A->nnz) {
            AUX_CUDA(cudaMemcpyAsync(col.p, A->col_idx, sizeof(int) * A->nnz, cudaMemcpyHostToDevice, h->stream));
            AUX_CUDA(cudaMemcpyAsync(v.p, A->values, sizeof(double) * A->nnz, cudaMemcpyHostToDevice, side.s));
        }
        AUX_CUDA(cudaEventRecord(side.e, side.s));
        aux_csr_view dv = *A;
        dv.row_ptr = rp.p;
        dv.col_idx = col.p;
        dv.values = v.p;
        setup_device(h, &dv, xy_d.p, (long)n_points, side.e);
        h->host_rp = A->row_ptr;
        h->host_col = A->col_idx;
        h->host_val = A->values;
        h->host_nnz = A->nnz;
        h->host_fp = csr_fingerprint(A);
        h->last_setup_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    });
    if (st != AUX_OK) {
        delete h;
        return st;
    }
    *out = h;
    return AUX_OK;
}

// ---- multi-GPU
void* aux_local_group_create(int32_t parts) {
    try {
        return local_group_create(parts);
    } catch (...) {
        return nullptr;
    }
}
void aux_local_group_destroy(void* g) { local_group_destroy(static_cast<LocalGroup*>(g)); }
int32_t aux_nccl_unique_id(uint8_t id[128]) { return nccl_unique_id(id) ? 1 : 0; }
void* aux_comm_create_nccl(const uint8_t id[128], int32_t nranks, int32_t rank, int32_t device) {
    try {
        DeviceGuard dg(device);
        return make_nccl_comm(id, nranks, rank);
    } catch (...) {
        return nullptr;
    }
}
void aux_comm_destroy(void* comm) { delete static_cast<Comm*>(comm); }

static aux_status setup_dist_impl(const aux_csr_view* A, const double* xy, int64_t n_points,
                                  const aux_setup_opts* opts, const aux_gpu_opts* gpu, const aux_dist_opts* d,
                                  aux_hierarchy** out, char* msg, size_t msg_len, bool host) {
    *out = nullptr;
    aux_hierarchy* h = nullptr;
    const aux_status st = guarded(msg, msg_len, [&] {
        if (!d || d->nparts < 1 || d->rank < 0 || d->rank >= d->nparts)
            throw_aux(AUX_ARGUMENT_ERROR, "aux_dist_opts: bad part count or rank");
        if (d->transport < 0 || d->transport > 2)
            throw_aux(AUX_ARGUMENT_ERROR, "aux_dist_opts: transport must be 0 (local), 1 (NCCL id) or 2 (communicator)");
        DeviceGuard dg(gpu ? gpu->device : 0);
        h = make_h(opts, gpu);
        const auto t0 = std::chrono::steady_clock::now();
        if (d->transport == 0) {
            if (!d->local_group || !is_local_group(d->local_group))
                throw_aux(AUX_ARGUMENT_ERROR, "aux_dist_opts: local transport needs a group (aux_local_group_create)");
            h->dist.comm = make_local_comm(static_cast<LocalGroup*>(d->local_group), d->rank);
        } else if (d->transport == 2) {
            if (!d->local_group || !is_comm(d->local_group))
                throw_aux(AUX_ARGUMENT_ERROR, "aux_dist_opts: transport 2 needs a communicator (aux_comm_create_nccl)");
            h->dist.comm = static_cast<Comm*>(d->local_group);
            h->dist.owns_comm = false;
            if (h->dist.comm->size != d->nparts || h->dist.comm->rank != d->rank)
                throw_aux(AUX_ARGUMENT_ERROR, "aux_dist_opts: communicator does not match nparts / rank");
        } else {
            h->dist.comm = make_nccl_comm(d->nccl_id, d->nparts, d->rank);
        }
        h->dist.dsum.alloc(8);
        if (A->n_rows < 0 || A->nnz < 0) throw_aux(AUX_SIZE_ERROR, "setup_hierarchy: negative size");
        if (host) {
            const long n = A->n_rows;
            DBuf<int> rp(n + 1), col(std::max<long>(A->nnz, 1));
            DBuf<double> v(std::max<long>(A->nnz, 1)), xy_d(2 * std::max<long>(n_points, 1));
            AUX_CUDA(cudaMemcpyAsync(rp.p, A->row_ptr, sizeof(int) * (n + 1), cudaMemcpyHostToDevice, h->stream));
            if (A->nnz) {
                AUX_CUDA(cudaMemcpyAsync(col.p, A->col_idx, sizeof(int) * A->nnz, cudaMemcpyHostToDevice, h->stream));
                AUX_CUDA(cudaMemcpyAsync(v.p, A->values, sizeof(double) * A->nnz, cudaMemcpyHostToDevice, h->stream));
            }
            if (n_points > 0)
                AUX_CUDA(cudaMemcpyAsync(xy_d.p, xy, sizeof(double) * 2 * n_points, cudaMemcpyHostToDevice, h->stream));
            aux_csr_view dv = *A;
            dv.row_ptr = rp.p;
            dv.col_idx = col.p;
            dv.values = v.p;
            setup_device_dist(h, &dv, xy_d.p, (long)n_points);
            h->host_rp = A->row_ptr;
            h->host_col = A->col_idx;
            h->host_val = A->values;
            h->host_nnz = A->nnz;
            h->host_fp = csr_fingerprint(A);
        } else {
            setup_device_dist(h, A, xy, (long)n_points);
        }
        h->last_setup_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    });
    if (st != AUX_OK) {
        delete h;
        return st;
    }
    *out = h;
    return AUX_OK;
}

aux_status aux_setup_dist(const aux_csr_view* A, const double* xy, int64_t n_points, const aux_setup_opts* opts,
                          const aux_gpu_opts* gpu, const aux_dist_opts* d, aux_hierarchy** out, char* msg,
                          size_t msg_len) {
    return setup_dist_impl(A, xy, n_points, opts, gpu, d, out, msg, msg_len, true);
}
aux_status aux_setup_dist_device(const aux_csr_view* A, const double* xy, int64_t n_points,
                                 const aux_setup_opts* opts, const aux_gpu_opts* gpu, const aux_dist_opts* d,
                                 aux_hierarchy** out, char* msg, size_t msg_len) {
    return setup_dist_impl(A, xy, n_points, opts, gpu, d, out, msg, msg_len, false);
}
int32_t aux_part_rows(const aux_hierarchy* h) { return h->fine.n; }
aux_status aux_part_dofs(const aux_hierarchy* h, int32_t* ids) {
    return guarded(nullptr, 0, [&] {
        DeviceGuard dg(h->gpu.device);
        const int32_t* src = h->dist.comm ? h->dist.gid.p : h->fine.perm.p;
        AUX_CUDA(cudaMemcpy(ids, src, sizeof(int32_t) * h->fine.n, cudaMemcpyDeviceToHost));
    });
}

aux_status aux_solve(aux_hierarchy* h, const aux_csr_view* A, const double* b, int64_t n_b,
                     const aux_cycle_opts* opts, aux_solve_result* res, char* msg, size_t msg_len) {
    return guarded(msg, msg_len, [&] {
        DeviceGuard dg(h->gpu.device);
        const auto t0 = std::chrono::steady_clock::now();
        aux_cycle_opts o;
        aux_default_cycle_opts(&o);
        if (opts) o = *opts;
        if (o.n_inner < 1 || o.pre_sweeps < 1 || o.post_sweeps < 1 || o.max_outer < 1)
            throw_aux(AUX_ARGUMENT_ERROR, "cycle options must be positive");
        if (!(o.rtol > 0.0) || !(o.rtol < 1.0)) throw_aux(AUX_ARGUMENT_ERROR, "rtol must lie in (0,1)");
        if (o.max_directions < 0) throw_aux(AUX_ARGUMENT_ERROR, "max_directions must be >= 0");
        h->outer = false;
        if (A) {
            if (n_b != A->n_rows) throw_aux(AUX_SIZE_ERROR, "solve: right-hand side does not match matrix");
            if (A->n_rows != h->n) throw_aux(AUX_SIZE_ERROR, "solve: hierarchy was built for a different order");
            // the setup matrix (same arrays, same sampled contents) reuses the
            // device copy; any other matrix is uploaded for the outer A z
            const bool same = A->row_ptr == h->host_rp && A->col_idx == h->host_col && A->values == h->host_val &&
                              A->nnz == h->host_nnz && csr_fingerprint(A) == h->host_fp;
            if (!same) set_outer_matrix(h, A);
        }
        const long n = h->n;
        DBuf<double> bd(std::max<long>(n_b, 1)), ud(std::max<long>(n, 1));
        if (n_b > 0)
            AUX_CUDA(cudaMemcpyAsync(bd.p, b, sizeof(double) * n_b, cudaMemcpyHostToDevice, h->stream));
        solve_device(h, bd.p, (long)n_b, &o, res, ud.p);
        if (res->u && n > 0 && h->dist.comm) {   // a part writes the entries of the DoFs it owns
            const long m = h->fine.n;
            if (m == n) {   // one part owns every DoF: u is already in caller order
                AUX_CUDA(cudaMemcpyAsync(res->u, ud.p, sizeof(double) * n, cudaMemcpyDeviceToHost, h->stream));
                AUX_CUDA(cudaStreamSynchronize(h->stream));
            } else if (m > 0) {   // owned entries in ascending caller id, copied run by run
                const std::vector<int>& runs = owned_runs(h);
                double* uv = pinned_scratch((size_t)m);
                gather_owned_sorted(h, ud.p, uv);
                AUX_CUDA(cudaStreamSynchronize(h->stream));
                for (size_t k = 0; k < runs.size(); k += 3)
                    std::memcpy(res->u + runs[k], uv + runs[k + 1], sizeof(double) * (size_t)runs[k + 2]);
            }
        } else if (res->u && n > 0) {
            AUX_CUDA(cudaMemcpyAsync(res->u, ud.p, sizeof(double) * n, cudaMemcpyDeviceToHost, h->stream));
            AUX_CUDA(cudaStreamSynchronize(h->stream));
        }
        const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        res->solve_seconds = secs;
        res->total_seconds = secs;
    });
}

aux_status aux_solve_device(aux_hierarchy* h, const double* b, int64_t n_b, const aux_cycle_opts* opts,
                            aux_solve_result* res, char* msg, size_t msg_len) {
    return guarded(msg, msg_len, [&] {
        DeviceGuard dg(h->gpu.device);
        aux_cycle_opts o;
        aux_default_cycle_opts(&o);
        if (opts) o = *opts;
        h->outer = false;
        solve_device(h, b, (long)n_b, &o, res, res->u);
    });
}

aux_status aux_stats(const aux_hierarchy* h, aux_stats_out* s) {
    std::memset(s, 0, sizeof *s);
    s->levels = (int32_t)h->lv.size();
    long total = 0;
    for (size_t i = 0; i < h->lv.size() && i < AUX_MAX_LEVELS; ++i) {
        s->sizes[i] = h->lv[i].n;
        s->nnz[i] = h->lv[i].nnz;
        total += h->lv[i].nnz;
    }
    s->operator_complexity = (double)total / (double)h->lv[0].nnz;
    return AUX_OK;
}

aux_status aux_get_locality(const aux_hierarchy* h, aux_locality* out) {
    *out = h->loc;
    return AUX_OK;
}

aux_status aux_grid(const aux_hierarchy* h, double box[4], int32_t* depth) {
    for (int i = 0; i < 4; ++i) box[i] = h->box[i];
    *depth = h->depth;
    return AUX_OK;
}

int32_t aux_n_levels(const aux_hierarchy* h) { return (int32_t)h->lv.size(); }

aux_status aux_level_info_get(const aux_hierarchy* h, int32_t level, aux_level_info* out) {
    if (level < 0 || level >= (int)h->lv.size()) return AUX_ARGUMENT_ERROR;
    return guarded(nullptr, 0, [&] {
        DeviceGuard dg(h->gpu.device);
        level_info(h, level, out);
    });
}

aux_status aux_export_level(const aux_hierarchy* h, int32_t level, aux_level_export* out) {
    if (level < 0 || level >= (int)h->lv.size() || h->dist.comm) return AUX_ARGUMENT_ERROR;
    return guarded(nullptr, 0, [&] {
        DeviceGuard dg(h->gpu.device);
        export_level(h, level, out);
    });
}

aux_status aux_export_coarsest(const aux_hierarchy* h, int32_t* n, double* lu, int32_t* perm) {
    return guarded(nullptr, 0, [&] {
        DeviceGuard dg(h->gpu.device);
        int nn = 0;
        export_coarsest(h, &nn, lu, perm);
        *n = nn;
    });
}

void aux_destroy(aux_hierarchy* h) {
    if (!h) return;
    const int dev = h->gpu.device;   // the buffers and the stream live there
    int prev = -1;
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
    delete h;
    if (prev >= 0 && prev != dev) cudaSetDevice(prev);
}

int64_t aux_launch_count(void) { return g_launches; }

void aux_profile_enable(aux_hierarchy* h, int32_t on) {
    h->prof.on = on < 0 ? 0 : (on > 2 ? 2 : on);
    h->graph_valid = false;   // mode 2 runs the coarse cycle eagerly; mode 0/1 recapture
    for (int k = 0; k < kProfKinds; ++k) {
        h->prof.used[k] = 0;
        h->prof.bytes[k] = 0;
        h->prof.launches[k] = 0;
        h->prof.total_ms[k] = 0;
    }
}

aux_status aux_profile_read(const aux_hierarchy* hc, int32_t kind, int64_t* launches, double* total_ms,
                            double* bytes_per_launch) {
    if (kind < 0 || kind >= kProfKinds) return AUX_ARGUMENT_ERROR;
    auto* h = const_cast<aux_hierarchy*>(hc);
    return guarded(nullptr, 0, [&] {
        DeviceGuard dg(h->gpu.device);
        AUX_CUDA(cudaStreamSynchronize(h->stream));
        Profile& P = h->prof;
        double ms = 0.0;
        for (size_t i = 0; i < P.used[kind]; ++i) {
            float t = 0.f;
            AUX_CUDA(cudaEventElapsedTime(&t, P.ev_begin[kind][i], P.ev_end[kind][i]));
            ms += t;
        }
        *launches = P.launches[kind];
        *total_ms = ms;
        *bytes_per_launch = P.launches[kind] ? P.bytes[kind] / (double)P.launches[kind] : 0.0;
    });
}

aux_status aux_last_timing(const aux_hierarchy* h, double* setup_ms, double* solve_ms) {
    *setup_ms = h->last_setup_ms;
    *solve_ms = h->last_solve_ms;
    return AUX_OK;
}

}  // extern "C"

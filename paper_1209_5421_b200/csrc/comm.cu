// comm.cu — CommLocal (P parts, one process, one device) and CommNccl.
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>

#include <mutex>
#include <set>

#include "comm.cuh"
#include "hier.cuh"

namespace auxb200 {

namespace {

__global__ void k_sum_parts(const double* __restrict__ slots, int parts, int cap, int count, double* __restrict__ out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
        double s = slots[i];
        for (int p = 1; p < parts; ++p) s += slots[(size_t)p * cap + i];
        out[i] = s;
    }
}
__global__ void k_max_parts(const unsigned long long* __restrict__ slots, int parts, int cap, int count,
                            unsigned long long* __restrict__ out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
        unsigned long long m = slots[i];
        for (int p = 1; p < parts; ++p) m = max(m, slots[(size_t)p * cap + i]);
        out[i] = m;
    }
}

// generation barrier for P host threads
struct HostBarrier {
    std::mutex m;
    std::condition_variable cv;
    int n, count = 0;
    long gen = 0;
    explicit HostBarrier(int parts) : n(parts) {}
    void wait() {
        std::unique_lock<std::mutex> lk(m);
        const long g = gen;
        if (++count == n) {
            count = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};

}  // namespace

struct LocalGroup {
    int P;
    HostBarrier bar;
    std::vector<const void*> box;     // [src * P + dst]
    std::vector<size_t> box_bytes;
    std::vector<cudaEvent_t> ready, done;
    DBuf<double> red;                 // [P][kRedCap]
    static constexpr int kRedCap = 64;
    explicit LocalGroup(int parts) : P(parts), bar(parts), box((size_t)parts * parts, nullptr),
                                     box_bytes((size_t)parts * parts, 0), ready(parts), done(parts) {
        for (int i = 0; i < P; ++i) {
            AUX_CUDA(cudaEventCreateWithFlags(&ready[i], cudaEventDisableTiming));
            AUX_CUDA(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming));
        }
        red.alloc((size_t)P * kRedCap);
    }
    ~LocalGroup() {
        for (int i = 0; i < P; ++i) {
            cudaEventDestroy(ready[i]);
            cudaEventDestroy(done[i]);
        }
    }
};

namespace {
std::mutex g_reg_mu;
std::set<const void*> g_groups, g_comms;
}  // namespace

bool is_local_group(const void* p) {
    std::lock_guard<std::mutex> lk(g_reg_mu);
    return g_groups.count(p) != 0;
}
bool is_comm(const void* p) {
    std::lock_guard<std::mutex> lk(g_reg_mu);
    return g_comms.count(p) != 0;
}
Comm::Comm() {
    std::lock_guard<std::mutex> lk(g_reg_mu);
    g_comms.insert(this);
}
Comm::~Comm() {
    std::lock_guard<std::mutex> lk(g_reg_mu);
    g_comms.erase(this);
}

LocalGroup* local_group_create(int parts) {
    if (parts < 1 || parts > 64) throw_aux(AUX_ARGUMENT_ERROR, "local group: 1..64 parts");
    LocalGroup* g = new LocalGroup(parts);
    std::lock_guard<std::mutex> lk(g_reg_mu);
    g_groups.insert(g);
    return g;
}
void local_group_destroy(LocalGroup* g) {
    {
        std::lock_guard<std::mutex> lk(g_reg_mu);
        g_groups.erase(g);
    }
    delete g;
}

namespace {

struct CommLocal : Comm {
    LocalGroup* g;
    CommLocal(LocalGroup* grp, int r) : g(grp) {
        rank = r;
        size = grp->P;
    }
    // phase 1: publish + ready event; barrier; phase 2: consume; done event; barrier;
    // then order later writes to my buffers after every consumer's copy
    void exchange(const std::vector<Msg>& sends, const std::vector<Msg>& recvs, cudaStream_t s) override {
        const int P = g->P;
        for (const Msg& m : sends) {
            g->box[(size_t)rank * P + m.peer] = m.buf;
            g->box_bytes[(size_t)rank * P + m.peer] = m.bytes;
        }
        AUX_CUDA(cudaEventRecord(g->ready[rank], s));
        g->bar.wait();
        for (const Msg& m : recvs) {
            const size_t k = (size_t)m.peer * P + rank;
            if (g->box_bytes[k] != m.bytes)
                throw_aux(AUX_INTERNAL_ERROR, "local exchange: message size mismatch from part " +
                                                  std::to_string(m.peer));
            AUX_CUDA(cudaStreamWaitEvent(s, g->ready[m.peer], 0));
            if (m.bytes) AUX_CUDA(cudaMemcpyAsync(m.buf, g->box[k], m.bytes, cudaMemcpyDeviceToDevice, s));
        }
        AUX_CUDA(cudaEventRecord(g->done[rank], s));
        g->bar.wait();
        // every mailbox read happened before the second barrier; later writes
        // to my send buffers wait for the consumers' copies
        for (const Msg& m : sends) AUX_CUDA(cudaStreamWaitEvent(s, g->done[m.peer], 0));
    }
    template <class T, class K>
    void reduce(T* buf, int count, cudaStream_t s, K kernel) {
        if (count > LocalGroup::kRedCap) throw_aux(AUX_INTERNAL_ERROR, "local allreduce: count too large");
        T* slots = reinterpret_cast<T*>(g->red.p);
        AUX_CUDA(cudaMemcpyAsync(slots + (size_t)rank * LocalGroup::kRedCap, buf, sizeof(T) * count,
                                 cudaMemcpyDeviceToDevice, s));
        AUX_CUDA(cudaEventRecord(g->ready[rank], s));
        g->bar.wait();
        for (int p = 0; p < g->P; ++p) AUX_CUDA(cudaStreamWaitEvent(s, g->ready[p], 0));
        kernel<<<1, 64, 0, s>>>(slots, g->P, LocalGroup::kRedCap, count, buf);
        AUX_CUDA(cudaEventRecord(g->done[rank], s));
        g->bar.wait();
        for (int p = 0; p < g->P; ++p) AUX_CUDA(cudaStreamWaitEvent(s, g->done[p], 0));
    }
    void allreduce_sum(double* buf, int count, cudaStream_t s) override {
        if (g->P > 1) reduce(buf, count, s, k_sum_parts);
    }
    void allreduce_max(unsigned long long* buf, int count, cudaStream_t s) override {
        if (g->P > 1) reduce(buf, count, s, k_max_parts);
    }
    void barrier(cudaStream_t s) override {
        AUX_CUDA(cudaStreamSynchronize(s));
        g->bar.wait();
    }
    bool graph_capturable() const override { return false; }   // host barriers between the parts
};

// ---- NCCL through dlopen (the process may already hold torch's libnccl)
struct NcclApi {
    bool ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!lib) return a;
#define AUX_SYM(f, name) a.f = reinterpret_cast<decltype(a.f)>(dlsym(lib, name))
        AUX_SYM(GetUniqueId, "ncclGetUniqueId");
        AUX_SYM(CommInitRank, "ncclCommInitRank");
        AUX_SYM(CommDestroy, "ncclCommDestroy");
        AUX_SYM(AllReduce, "ncclAllReduce");
        AUX_SYM(Send, "ncclSend");
        AUX_SYM(Recv, "ncclRecv");
        AUX_SYM(GroupStart, "ncclGroupStart");
        AUX_SYM(GroupEnd, "ncclGroupEnd");
        AUX_SYM(GetErrorString, "ncclGetErrorString");
#undef AUX_SYM
        a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.AllReduce && a.Send && a.Recv && a.GroupStart &&
               a.GroupEnd && a.GetErrorString;
        return a;
    }();
    return api;
}

#define AUX_NCCL(call)                                                                             \
    do {                                                                                           \
        ncclResult_t r_ = (call);                                                                  \
        if (r_ != ncclSuccess)                                                                     \
            throw_aux(AUX_CUDA_ERROR, std::string("NCCL: ") + #call + ": " + nccl().GetErrorString(r_)); \
    } while (0)

struct CommNccl : Comm {
    ncclComm_t comm = nullptr;
    CommNccl(const unsigned char id[128], int n, int r) {
        rank = r;
        size = n;
        if (!nccl().ok) throw_aux(AUX_CUDA_ERROR, "libnccl.so.2 not found");
        ncclUniqueId uid;
        std::memcpy(uid.internal, id, sizeof uid.internal);
        AUX_NCCL(nccl().CommInitRank(&comm, n, uid, r));
    }
    ~CommNccl() override {
        if (comm) nccl().CommDestroy(comm);
    }
    void allreduce_sum(double* buf, int count, cudaStream_t s) override {
        if (size > 1) AUX_NCCL(nccl().AllReduce(buf, buf, count, ncclFloat64, ncclSum, comm, s));
    }
    void allreduce_max(unsigned long long* buf, int count, cudaStream_t s) override {
        if (size > 1) AUX_NCCL(nccl().AllReduce(buf, buf, count, ncclUint64, ncclMax, comm, s));
    }
    void exchange(const std::vector<Msg>& sends, const std::vector<Msg>& recvs, cudaStream_t s) override {
        if (sends.empty() && recvs.empty()) return;
        AUX_NCCL(nccl().GroupStart());
        for (const Msg& m : sends)
            if (m.bytes) AUX_NCCL(nccl().Send(m.buf, m.bytes, ncclUint8, m.peer, comm, s));
        for (const Msg& m : recvs)
            if (m.bytes) AUX_NCCL(nccl().Recv(m.buf, m.bytes, ncclUint8, m.peer, comm, s));
        AUX_NCCL(nccl().GroupEnd());
    }
    bool graph_capturable() const override { return true; }   // NCCL kernels capture into CUDA graphs
    void barrier(cudaStream_t s) override {
        DBuf<double> one(1);
        AUX_CUDA(cudaMemsetAsync(one.p, 0, sizeof(double), s));
        allreduce_sum(one.p, 1, s);
        AUX_CUDA(cudaStreamSynchronize(s));
    }
};

}  // namespace

Comm* make_local_comm(LocalGroup* g, int rank) {
    if (!g || rank < 0 || rank >= g->P) throw_aux(AUX_ARGUMENT_ERROR, "local comm: bad rank");
    return new CommLocal(g, rank);
}

bool nccl_unique_id(unsigned char id[128]) {
    if (!nccl().ok) return false;
    ncclUniqueId uid;
    if (nccl().GetUniqueId(&uid) != ncclSuccess) return false;
    std::memcpy(id, uid.internal, 128);
    return true;
}

Comm* make_nccl_comm(const unsigned char id[128], int nranks, int rank) { return new CommNccl(id, nranks, rank); }

}  // namespace auxb200

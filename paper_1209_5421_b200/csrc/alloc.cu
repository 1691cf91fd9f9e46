// alloc.cu — process-wide caching device allocator (see hier.cuh).
#include <condition_variable>
#include <thread>
#include <cstdlib>
#include <map>
#include <mutex>
#include <set>
#include <tuple>
#include <vector>

#include "hier.cuh"

namespace auxb200 {

namespace {

// One cache per host thread: a block freed while kernels of its stream may
// still use it is only handed out again to the same thread, whose work is
// ordered on that stream (or synchronised before it moves to another one:
// setup and solve end with a stream synchronisation, a hierarchy synchronises
// before releasing its buffers).  The multi-part test transport drives one
// part per thread, each on its own stream.
std::mutex g_mu;   // guards cudaMalloc / cudaFree of the retry path
// Blocks are keyed by (device, rounded size): a block is only handed to a
// request on the device it was allocated on.
using Key = std::pair<int, size_t>;
struct Cache {
    std::multimap<Key, void*> m;   // (device, rounded size) -> cached block
    ~Cache() {   // thread exit: the blocks go back to the driver
        for (auto& kv : m) cudaFree(kv.second);
    }
    auto find(const Key& r) { return m.find(r); }
    auto end() { return m.end(); }
    void erase(std::multimap<Key, void*>::iterator it) { m.erase(it); }
    void emplace(const Key& r, void* p) { m.emplace(r, p); }
    void clear(int dev) {   // the current device's blocks
        for (auto it = m.begin(); it != m.end();) {
            if (it->first.first == dev) {
                cudaFree(it->second);
                it = m.erase(it);
            } else {
                ++it;
            }
        }
    }
};
thread_local Cache g_free;

size_t round_size(size_t b) {
    if (b <= 512) return 512;
    if (b <= (size_t(64) << 20)) {
        size_t r = 512;
        while (r < b) r <<= 1;
        return r;
    }
    const size_t g = size_t(64) << 20;
    return (b + g - 1) / g * g;
}

}  // namespace

int current_device() {
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess) d = 0;
    return d;
}

void* dev_alloc(size_t bytes) {
    const int dev = current_device();
    const size_t r = round_size(bytes);
    {
        auto it = g_free.find(Key{dev, r});
        if (it != g_free.end()) {
            void* p = it->second;
            g_free.erase(it);
            return p;
        }
    }
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, r);
    if (e != cudaSuccess) {
        // release the cache and retry once
        (void)cudaGetLastError();
        std::lock_guard<std::mutex> lk(g_mu);
        cudaDeviceSynchronize();
        g_free.clear(dev);
        e = cudaMalloc(&p, r);
    }
    if (e != cudaSuccess) throw_aux(AUX_CUDA_ERROR, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    return p;
}

void dev_free(void* p, size_t bytes) {
    if (!p) return;
    cudaPointerAttributes at{};
    const int dev = cudaPointerGetAttributes(&at, p) == cudaSuccess ? at.device : current_device();
    g_free.emplace(Key{dev, round_size(bytes)}, p);
}

void ensure_smem_impl(const void* func, int bytes) {
    static std::mutex mu;
    static std::set<std::tuple<const void*, int, int>> done;
    const int dev = current_device();
    std::lock_guard<std::mutex> lk(mu);
    if (done.count({func, dev, bytes})) return;
    AUX_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    done.insert({func, dev, bytes});
}

namespace {
struct DriverPools {
    std::mutex mu;
    std::multimap<int, cudaStream_t> streams;    // device -> idle stream
};
DriverPools& pools() {
    static DriverPools* p = new DriverPools();   // never destroyed: outlives every hierarchy
    return *p;
}
}  // namespace

cudaStream_t stream_pool_get() {
    const int dev = current_device();
    {
        std::lock_guard<std::mutex> lk(pools().mu);
        auto it = pools().streams.find(dev);
        if (it != pools().streams.end()) {
            cudaStream_t s = it->second;
            pools().streams.erase(it);
            return s;
        }
    }
    cudaStream_t s = nullptr;
    AUX_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    return s;
}

void stream_pool_put(cudaStream_t s) {   // the caller synchronised it
    if (!s) return;
    const int dev = current_device();
    std::lock_guard<std::mutex> lk(pools().mu);
    pools().streams.emplace(dev, s);
}

// A retired executable graph is destroyed by a background thread: the
// destroy call blocks for 10+ ms whenever another process holds the driver
// lock, and nothing waits for it.  (Re-targeting cached executables with
// cudaGraphExecUpdate was tried: the update reports success for captures of
// another hierarchy with the same topology, yet the replay is wrong.)
cudaGraphExec_t graph_exec_acquire(cudaGraph_t g) {
    cudaGraphExec_t e = nullptr;
    AUX_CUDA(cudaGraphInstantiate(&e, g, 0));
    return e;
}

namespace {
struct Reaper {
    std::mutex mu;
    std::mutex busy;   // held while destroying: process exit waits for the batch, then stops the thread
    std::condition_variable cv;
    std::vector<std::pair<int, cudaGraphExec_t>> q;
    bool started = false;
    bool exiting = false;
    void start() {
        std::atexit([] {   // before the CUDA runtime's own teardown; leftovers go with the context
            Reaper& r = reaper_ref();
            {
                std::lock_guard<std::mutex> lk(r.mu);
                r.exiting = true;
                r.cv.notify_one();
            }
            std::lock_guard<std::mutex> b(r.busy);   // a batch in progress finishes first
        });
        std::thread([this] {
            for (;;) {
                std::vector<std::pair<int, cudaGraphExec_t>> work;
                std::unique_lock<std::mutex> b(busy, std::defer_lock);
                {
                    std::unique_lock<std::mutex> lk(mu);
                    cv.wait(lk, [this] { return !q.empty() || exiting; });
                    if (exiting) return;
                    work.swap(q);
                    b.lock();   // (taken under mu: exit either sees no batch or waits for this one)
                }
                for (auto& w : work) {
                    cudaSetDevice(w.first);
                    cudaGraphExecDestroy(w.second);
                }
            }
        }).detach();
    }
    static Reaper& reaper_ref();
};
Reaper& Reaper::reaper_ref() {
    static Reaper* r = new Reaper();   // never destroyed (detached thread)
    return *r;
}
Reaper& reaper() { return Reaper::reaper_ref(); }
}  // namespace

void graph_exec_release(cudaGraphExec_t e) {   // no launch of e may still be in flight
    if (!e) return;
    Reaper& r = reaper();
    std::lock_guard<std::mutex> lk(r.mu);
    if (!r.started) {
        r.start();
        r.started = true;
    }
    if (r.exiting) return;   // the context goes away with the process
    r.q.emplace_back(current_device(), e);
    r.cv.notify_one();
}

}  // namespace auxb200

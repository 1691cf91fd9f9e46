// alloc.cu — process-wide caching device allocator (see hier.cuh).
#include <map>
#include <mutex>
#include <set>
#include <tuple>

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

}  // namespace auxb200

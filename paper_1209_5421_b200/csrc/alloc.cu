// alloc.cu — process-wide caching device allocator (see hier.cuh).
#include <map>
#include <mutex>

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
struct Cache {
    std::multimap<size_t, void*> m;   // rounded size -> cached block
    ~Cache() {   // thread exit: the blocks go back to the driver
        for (auto& kv : m) cudaFree(kv.second);
    }
    auto find(size_t r) { return m.find(r); }
    auto end() { return m.end(); }
    void erase(std::multimap<size_t, void*>::iterator it) { m.erase(it); }
    void emplace(size_t r, void* p) { m.emplace(r, p); }
    void clear() {
        for (auto& kv : m) cudaFree(kv.second);
        m.clear();
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

void* dev_alloc(size_t bytes) {
    const size_t r = round_size(bytes);
    {
        auto it = g_free.find(r);
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
        g_free.clear();
        e = cudaMalloc(&p, r);
    }
    if (e != cudaSuccess) throw_aux(AUX_CUDA_ERROR, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    return p;
}

void dev_free(void* p, size_t bytes) {
    if (!p) return;
    g_free.emplace(round_size(bytes), p);
}

}  // namespace auxb200

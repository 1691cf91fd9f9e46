// alloc.cu — process-wide caching device allocator (see hier.cuh).
#include <map>
#include <mutex>

#include "hier.cuh"

namespace auxb200 {

namespace {

std::mutex g_mu;
std::multimap<size_t, void*> g_free;   // rounded size -> cached block

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
        std::lock_guard<std::mutex> lk(g_mu);
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
        for (auto& kv : g_free) cudaFree(kv.second);
        g_free.clear();
        e = cudaMalloc(&p, r);
    }
    if (e != cudaSuccess) throw_aux(AUX_CUDA_ERROR, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    return p;
}

void dev_free(void* p, size_t bytes) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(g_mu);
    g_free.emplace(round_size(bytes), p);
}

}  // namespace auxb200

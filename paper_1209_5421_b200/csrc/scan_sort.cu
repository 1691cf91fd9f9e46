// scan_sort.cu — device-wide exclusive scan and stable LSD radix sort.
//
// The radix sort replaces the reference's counting sort in build_members
// (auxgrid.hpp:58-70): sorting (cell key, DoF id) pairs stably by key leaves
// the DoFs of every cell in ascending id order, exactly the member order of
// the reference, so member_idx is bitwise identical.  8-bit digits, 4096-key
// tiles; ranks inside a tile come from warp match masks, so the sort is
// deterministic and stable.
#include "scan_sort.cuh"

namespace auxb200 {

namespace {

constexpr int kScanThreads = 256;
constexpr int kScanPer = 8;
constexpr int kScanTile = kScanThreads * kScanPer;   // 2048

__global__ void k_scan_reduce(const int* __restrict__ in, long n, long long* __restrict__ bsum) {
    __shared__ long long sm[kScanThreads / 32];
    const long base = static_cast<long>(blockIdx.x) * kScanTile;
    long long s = 0;
    for (int i = threadIdx.x; i < kScanTile; i += kScanThreads) {
        const long j = base + i;
        if (j < n) s += in[j];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long t = 0;
        for (int w = 0; w < kScanThreads / 32; ++w) t += sm[w];
        bsum[blockIdx.x] = t;
    }
}

// Single-block exclusive scan of nb block sums (in place), total in bsum[nb].
__global__ void k_scan_bsums(long long* bsum, long nb) {
    __shared__ long long sm[1024];
    __shared__ long long carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (long base = 0; base < nb; base += 1024) {
        const long j = base + threadIdx.x;
        const long long v = j < nb ? bsum[j] : 0;
        sm[threadIdx.x] = v;
        __syncthreads();
        for (int o = 1; o < 1024; o <<= 1) {
            const long long t = threadIdx.x >= o ? sm[threadIdx.x - o] : 0;
            __syncthreads();
            sm[threadIdx.x] += t;
            __syncthreads();
        }
        if (j < nb) bsum[j] = carry + sm[threadIdx.x] - v;
        __syncthreads();
        if (threadIdx.x == 1023) carry += sm[1023];
        __syncthreads();
    }
    if (threadIdx.x == 0) bsum[nb] = carry;
}

__global__ void k_scan_final(const int* __restrict__ in, long n, const long long* __restrict__ bsum,
                             int* __restrict__ out) {
    __shared__ long long sm[kScanThreads];
    const long base = static_cast<long>(blockIdx.x) * kScanTile + static_cast<long>(threadIdx.x) * kScanPer;
    long long v[kScanPer];
    long long t = 0;
#pragma unroll
    for (int i = 0; i < kScanPer; ++i) {
        const long j = base + i;
        v[i] = j < n ? in[j] : 0;
        t += v[i];
    }
    sm[threadIdx.x] = t;
    __syncthreads();
    for (int o = 1; o < kScanThreads; o <<= 1) {
        const long long x = threadIdx.x >= o ? sm[threadIdx.x - o] : 0;
        __syncthreads();
        sm[threadIdx.x] += x;
        __syncthreads();
    }
    long long run = bsum[blockIdx.x] + sm[threadIdx.x] - t;
#pragma unroll
    for (int i = 0; i < kScanPer; ++i) {
        const long j = base + i;
        if (j < n) out[j] = static_cast<int>(run);
        run += v[i];
    }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) out[n] = static_cast<int>(bsum[gridDim.x]);
}

constexpr int kSortThreads = 256;
constexpr int kSortRounds = 16;
constexpr int kSortTile = kSortThreads * kSortRounds;   // 4096 keys

__global__ void k_rs_hist(const unsigned* __restrict__ keys, long n, int shift, int* __restrict__ hist,
                          int nblocks) {
    __shared__ int h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const long base = static_cast<long>(blockIdx.x) * kSortTile;
    for (int r = 0; r < kSortRounds; ++r) {
        const long i = base + r * kSortThreads + threadIdx.x;
        if (i < n) atomicAdd(&h[(keys[i] >> shift) & 255u], 1);
    }
    __syncthreads();
    hist[threadIdx.x * nblocks + blockIdx.x] = h[threadIdx.x];
}

__global__ void k_rs_scatter(const unsigned* __restrict__ kin, const int* __restrict__ vin,
                             unsigned* __restrict__ kout, int* __restrict__ vout, long n, int shift,
                             const int* __restrict__ offs, int nblocks) {
    __shared__ int base[256];
    __shared__ int wcnt[kSortThreads / 32][256];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    base[threadIdx.x] = offs[threadIdx.x * nblocks + blockIdx.x];
#pragma unroll
    for (int w = 0; w < kSortThreads / 32; ++w) wcnt[w][threadIdx.x] = 0;
    __syncthreads();
    const unsigned lt = (1u << lane) - 1u;
    const long tile = static_cast<long>(blockIdx.x) * kSortTile;
    for (int r = 0; r < kSortRounds; ++r) {
        const long i = tile + r * kSortThreads + threadIdx.x;
        const bool valid = i < n;
        unsigned key = 0;
        int val = 0;
        int d = 256;
        if (valid) {
            key = kin[i];
            val = vin[i];
            d = static_cast<int>((key >> shift) & 255u);
        }
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const int rank = __popc(peers & lt);
        if (valid && lane == __ffs(peers) - 1) wcnt[warp][d] = __popc(peers);
        __syncthreads();
        if (valid) {
            int off = base[d];
            for (int w = 0; w < warp; ++w) off += wcnt[w][d];
            kout[off + rank] = key;
            vout[off + rank] = val;
        }
        __syncthreads();
        int tot = 0;
#pragma unroll
        for (int w = 0; w < kSortThreads / 32; ++w) {
            tot += wcnt[w][threadIdx.x];
            wcnt[w][threadIdx.x] = 0;
        }
        base[threadIdx.x] += tot;
        __syncthreads();
    }
}

__global__ void k_iota(int* v, long n) {
    for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n; i += static_cast<long>(gridDim.x) * blockDim.x)
        v[i] = static_cast<int>(i);
}

}  // namespace

void exclusive_scan(const int* in, int* out, long n, cudaStream_t s) {
    const long nb = (n + kScanTile - 1) / kScanTile;
    if (nb == 0) {
        AUX_CUDA(cudaMemsetAsync(out, 0, sizeof(int), s));
        return;
    }
    DBuf<long long> bsum(static_cast<size_t>(nb) + 1);
    k_scan_reduce<<<static_cast<unsigned>(nb), kScanThreads, 0, s>>>(in, n, bsum.p);
    k_scan_bsums<<<1, 1024, 0, s>>>(bsum.p, nb);
    k_scan_final<<<static_cast<unsigned>(nb), kScanThreads, 0, s>>>(in, n, bsum.p, out);
    AUX_LAUNCHED(3);
    AUX_CUDA(cudaGetLastError());
    // no synchronisation: bsum goes back to this thread's allocator cache and
    // is only handed out again to work of this thread, ordered on its stream
    // (alloc.cu), so the scan stays asynchronous
}

void radix_sort_pairs(unsigned* keys, int* vals, long n, int nbits, cudaStream_t s, bool iota_vals) {
    if (n <= 0) return;
    if (iota_vals) {
        k_iota<<<592, 256, 0, s>>>(vals, n);
        AUX_LAUNCHED(1);
    }
    const int nblocks = static_cast<int>((n + kSortTile - 1) / kSortTile);
    DBuf<unsigned> k2(static_cast<size_t>(n));
    DBuf<int> v2(static_cast<size_t>(n));
    DBuf<int> hist(static_cast<size_t>(256) * nblocks);
    DBuf<int> offs(static_cast<size_t>(256) * nblocks + 1);
    unsigned *ka = keys, *kb = k2.p;
    int *va = vals, *vb = v2.p;
    int passes = 0;
    for (int shift = 0; shift < nbits; shift += 8, ++passes) {
        k_rs_hist<<<nblocks, kSortThreads, 0, s>>>(ka, n, shift, hist.p, nblocks);
        AUX_LAUNCHED(1);
        exclusive_scan(hist.p, offs.p, static_cast<long>(256) * nblocks, s);
        k_rs_scatter<<<nblocks, kSortThreads, 0, s>>>(ka, va, kb, vb, n, shift, offs.p, nblocks);
        AUX_LAUNCHED(1);
        AUX_CUDA(cudaGetLastError());
        std::swap(ka, kb);
        std::swap(va, vb);
    }
    if (passes % 2 == 1) {
        AUX_CUDA(cudaMemcpyAsync(keys, ka, sizeof(unsigned) * n, cudaMemcpyDeviceToDevice, s));
        AUX_CUDA(cudaMemcpyAsync(vals, va, sizeof(int) * n, cudaMemcpyDeviceToDevice, s));
    }
    // (scratch buffers return to the stream-ordered cache: no synchronisation)
}

}  // namespace auxb200

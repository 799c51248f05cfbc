// Calibration for the insert path (cache.cpp:94-119 update(): scan, then one
// compare-and-swap): random read-modify-write throughput of B200 HBM over an
// 800 MB buffer (the 1e7 x 10 table's size).
//   cas8      one 8-byte atomicCAS per access at a random 8-byte-aligned word
//             (the dirty line is written back on eviction: a read and a write
//             per access)
//   read64    one coalesced 64-byte read (4 lanes x 16 B) per access (the
//             probe's head read) -- the read-only ceiling, for comparison
//   read64cas one 64-byte read and then an 8-byte atomicCAS into the same
//             64 bytes (the probe + insert of an empty slot)
// Every lane keeps kInFlight independent accesses in flight; addresses come
// from a per-lane LCG reduced with a multiply-high. Prints accesses/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o rand_rmw rand_rmw.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

template <int kInFlight>
__global__ void __launch_bounds__(256) k_cas8(unsigned long long* buf, uint32_t n_words, uint32_t iters,
                                              unsigned long long* sink) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    uint64_t s = mix64(tid);
    unsigned long long acc = 0;
    for (uint32_t it = 0; it < iters; it += kInFlight) {
        unsigned long long v[kInFlight];
#pragma unroll
        for (int u = 0; u < kInFlight; ++u) {
            s = s * 6364136223846793005ull + 1442695040888963407ull;
            const uint32_t w = static_cast<uint32_t>(((s >> 32) * n_words) >> 32);
            v[u] = atomicCAS(buf + w, 0ull, s | 1ull);
        }
#pragma unroll
        for (int u = 0; u < kInFlight; ++u) acc += v[u];
    }
    if (acc == 0x1234567ull) atomicAdd(sink, acc);
}

// 4 adjacent lanes read one 64-byte block (16 B each); with kCas, the group's
// first lane then CASes one word of that block.
template <int kInFlight, bool kCas>
__global__ void __launch_bounds__(256) k_read64(uint4* buf, uint32_t n_blocks, uint32_t iters,
                                                unsigned long long* sink) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const int sub = threadIdx.x & 3;
    uint64_t s = mix64(tid >> 2);
    unsigned long long acc = 0;
    for (uint32_t it = 0; it < iters; it += kInFlight) {
        uint4 v[kInFlight];
        uint32_t blk[kInFlight];
#pragma unroll
        for (int u = 0; u < kInFlight; ++u) {
            s = s * 6364136223846793005ull + 1442695040888963407ull;
            blk[u] = static_cast<uint32_t>(((s >> 32) * n_blocks) >> 32);
            v[u] = __ldcg(buf + static_cast<uint64_t>(blk[u]) * 4 + sub);
        }
#pragma unroll
        for (int u = 0; u < kInFlight; ++u) {
            acc += v[u].x ^ v[u].w;
            if (kCas && sub == 0) {
                unsigned long long* w = reinterpret_cast<unsigned long long*>(buf + static_cast<uint64_t>(blk[u]) * 4);
                acc += atomicCAS(w + (v[u].y & 7u), 0ull, s | 1ull);
            }
        }
    }
    if (acc == 0x1234567ull) atomicAdd(sink, acc);
}

// The same access pattern written as rand_read2.cu's k_randw (byte pointer,
// a 32-bit fold per load): the form that reaches the ~44 G accesses/s
// random-read ceiling there.
template <bool kCas>
__global__ void __launch_bounds__(256) k_read64w(uint8_t* buf, uint32_t n_units, uint32_t iters,
                                                 unsigned long long* sink) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const int sub = (threadIdx.x & 31) % 4;
    const uint64_t group = tid / 4;
    uint64_t s = mix64(group);
    uint32_t acc = 0;
    for (uint32_t it = 0; it < iters; it += 4) {
        uint32_t v[4];
        uint8_t* p[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            s = s * 6364136223846793005ull + 1442695040888963407ull;
            const uint32_t unit = static_cast<uint32_t>(((s >> 32) * n_units) >> 32);
            p[u] = buf + static_cast<uint64_t>(unit) * 64;
            const uint4 t = __ldcg(reinterpret_cast<const uint4*>(p[u] + sub * 16));
            v[u] = t.x ^ t.y ^ t.z ^ t.w;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            acc += v[u];
            if (kCas && sub == 0) {
                acc += static_cast<uint32_t>(atomicCAS(reinterpret_cast<unsigned long long*>(p[u]) + (v[u] & 7u),
                                                       0ull, s | 1ull));
            }
        }
    }
    if (acc == 0x1234567u) atomicAdd(sink, acc);
}

int main() {
    const size_t bytes = 800000000ull;
    void* buf;
    unsigned long long* sink;
    cudaMalloc(&buf, bytes);
    cudaMalloc(&sink, 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int threads = 256;
    const uint32_t iters = 256;
    auto run = [&](const char* name, int bps, int lanes, int depth, auto launch) {
        const int blocks = sms * bps;
        cudaMemset(buf, 0, bytes);
        launch(blocks);   // warm-up (fills some words: CAS from 0 then fails -- still an RMW)
        cudaMemset(buf, 0, bytes);
        cudaDeviceSynchronize();
        cudaEventRecord(a);
        launch(blocks);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double accesses = (double)blocks * threads / lanes * iters;
        printf("{\"access\": \"%s\", \"in_flight\": %d, \"blocks_per_sm\": %d, \"ms\": %.3f, \"Gaccess_s\": %.2f}\n",
               name, depth, bps, ms, accesses / ms / 1e6);
    };
    unsigned long long* w = static_cast<unsigned long long*>(buf);
    uint4* q = static_cast<uint4*>(buf);
    for (int bps : {4, 8}) {
        run("cas8", bps, 1, 4, [&](int blocks) { k_cas8<4><<<blocks, threads>>>(w, (uint32_t)(bytes / 8), iters, sink); });
        run("cas8", bps, 1, 8, [&](int blocks) { k_cas8<8><<<blocks, threads>>>(w, (uint32_t)(bytes / 8), iters, sink); });
        run("read64", bps, 4, 4, [&](int blocks) { k_read64<4, false><<<blocks, threads>>>(q, (uint32_t)(bytes / 64), iters, sink); });
        run("read64cas", bps, 4, 4, [&](int blocks) { k_read64<4, true><<<blocks, threads>>>(q, (uint32_t)(bytes / 64), iters, sink); });
        run("read64cas", bps, 4, 8, [&](int blocks) { k_read64<8, true><<<blocks, threads>>>(q, (uint32_t)(bytes / 64), iters, sink); });
        run("read64w", bps, 4, 4, [&](int blocks) { k_read64w<false><<<blocks, threads>>>(static_cast<uint8_t*>(buf), (uint32_t)(bytes / 64), iters, sink); });
        run("read64w_cas", bps, 4, 4, [&](int blocks) { k_read64w<true><<<blocks, threads>>>(static_cast<uint8_t*>(buf), (uint32_t)(bytes / 64), iters, sink); });
    }
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    return 0;
}

// Calibration: random-access read throughput of B200 HBM at the granularities
// the cache probe uses, over an 800 MB buffer (the 1e7 x 10 table's size).
// For each access size S (16..128 B, S-aligned) a warp issues 32 random
// accesses; bandwidth = bytes requested / time. The ceiling this measures is
// what a random cell probe can reach, next to the copy peak.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o rand_read rand_read.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

// Each thread: `iters` random accesses of S bytes, loaded by S/16 lanes of a
// lane group (so one access = one coalesced request) -- kLanes lanes per access.
template <int kBytes>
__global__ void k_rand(const uint4* buf, uint64_t n_units, uint64_t iters, unsigned long long* sink) {
    constexpr int kLanes = kBytes / 16;  // 16 B per lane
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const int sub = lane % kLanes;
    const uint64_t group = tid / kLanes;
    uint64_t acc = 0;
    for (uint64_t it = 0; it < iters; it += 4) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint64_t h = mix64(group * 0x9e3779b97f4a7c15ull + it + u);
            v[u] = __ldcg(buf + (h % n_units) * kLanes + sub);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) acc += v[u].x ^ v[u].w;
    }
    if (acc == 0x1234567) atomicAdd(sink, acc);
}

// 80-byte cells at 80-byte stride (the table's layout), 5 lanes x 16 B.
__global__ void k_cells(const uint4* buf, uint64_t n_cells, uint64_t iters, unsigned long long* sink) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    if (lane >= 30) return;
    const int sub = lane % 5;
    const uint64_t group = (tid / 32) * 6 + lane / 5;
    uint64_t acc = 0;
    for (uint64_t it = 0; it < iters; it += 4) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint64_t cell = mix64(group * 0x9e3779b97f4a7c15ull + it + u) % n_cells;
            v[u] = __ldcg(buf + cell * 5 + sub);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) acc += v[u].x ^ v[u].w;
    }
    if (acc == 0x1234567) atomicAdd(sink, acc);
}

int main() {
    const size_t bytes = 800000000ull;
    uint4* buf;
    unsigned long long* sink;
    cudaMalloc(&buf, bytes);
    cudaMalloc(&sink, 8);
    cudaMemset(buf, 1, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int blocks = 148 * 8, threads = 256;
    const uint64_t iters = 256;
    auto run = [&](const char* name, auto launch, double bytes_per_access, double accesses) {
        launch();
        cudaEventRecord(a);
        launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("{\"access\": \"%s\", \"ms\": %.3f, \"GBps\": %.1f, \"Gaccess_s\": %.2f}\n", name, ms,
               accesses * bytes_per_access / ms / 1e6, accesses / ms / 1e6);
    };
    const double total_threads = (double)blocks * threads;
#define RUN(S)                                                                                   \
    run(#S "B", [&] { k_rand<S><<<blocks, threads>>>(buf, bytes / S, iters, sink); }, S,          \
        total_threads / (S / 16) * iters);
    RUN(16)
    RUN(32)
    RUN(64)
    RUN(128)
    run("80B-cell", [&] { k_cells<<<blocks, threads>>>(buf, bytes / 80, iters, sink); }, 80,
        (double)blocks * threads / 32 * 6 * iters);
    // sequential copy-style read for reference
    return 0;
}

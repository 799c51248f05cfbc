// Calibration v2: random-access read throughput of B200 HBM over an 800 MB
// buffer (the 1e7 x 10 table's size), at the granularities a cell probe can
// use. rand_read.cu reduced addresses with a 64-bit `%` (an emulated division:
// the kernel was issue-bound at ~23 G accesses/s whatever the size); here the
// range reduction is a multiply-high (Lemire), every thread keeps kInFlight
// independent accesses in flight, and an access of S bytes is one coalesced
// request of S/16 adjacent lanes. Prints accesses/s and bytes/s per size and
// per in-flight depth: the random-access ceiling the probe is compared with.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o rand_read2 rand_read2.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

template <int kBytes, int kInFlight>
__global__ void __launch_bounds__(256) k_rand(const uint4* buf, uint32_t n_units, uint32_t iters,
                                              unsigned long long* sink) {
    constexpr int kLanes = kBytes >= 16 ? kBytes / 16 : 1;
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const int sub = (threadIdx.x & 31) % kLanes;
    const uint64_t group = tid / kLanes;
    uint64_t s = mix64(group);
    uint32_t acc = 0;
    for (uint32_t it = 0; it < iters; it += kInFlight) {
        uint4 v[kInFlight];
#pragma unroll
        for (int u = 0; u < kInFlight; ++u) {
            s = s * 6364136223846793005ull + 1442695040888963407ull;   // LCG per group
            const uint32_t unit = static_cast<uint32_t>(((s >> 32) * n_units) >> 32);
            if (kBytes >= 16) {
                v[u] = __ldcg(buf + static_cast<uint64_t>(unit) * kLanes + sub);
            } else {
                const uint32_t* b32 = reinterpret_cast<const uint32_t*>(buf);
                v[u].x = __ldcg(b32 + static_cast<uint64_t>(unit) * (kBytes / 4));
                v[u].w = 0;
            }
        }
#pragma unroll
        for (int u = 0; u < kInFlight; ++u) acc += v[u].x ^ v[u].w;
    }
    if (acc == 0x1234567u) atomicAdd(sink, acc);
}

// Access of S bytes made by S/W adjacent lanes with W-byte loads (W = 4, 8,
// 16): does the load width change the random-access rate?
template <int S, int W>
__global__ void __launch_bounds__(256) k_randw(const uint8_t* buf, uint32_t n_units, uint32_t iters,
                                               unsigned long long* sink) {
    constexpr int kLanes = S / W;
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const int sub = (threadIdx.x & 31) % kLanes;
    const uint64_t group = tid / kLanes;
    uint64_t s = mix64(group);
    uint32_t acc = 0;
    for (uint32_t it = 0; it < iters; it += 4) {
        uint32_t v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            s = s * 6364136223846793005ull + 1442695040888963407ull;
            const uint32_t unit = static_cast<uint32_t>(((s >> 32) * n_units) >> 32);
            const uint8_t* p = buf + static_cast<uint64_t>(unit) * S + sub * W;
            if (W == 4) v[u] = __ldcg(reinterpret_cast<const uint32_t*>(p));
            else if (W == 8) { const uint2 t = __ldcg(reinterpret_cast<const uint2*>(p)); v[u] = t.x ^ t.y; }
            else { const uint4 t = __ldcg(reinterpret_cast<const uint4*>(p)); v[u] = t.x ^ t.y ^ t.z ^ t.w; }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) acc += v[u];
    }
    if (acc == 0x1234567u) atomicAdd(sink, acc);
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
    int dev = 0, sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int threads = 256;
    const uint32_t iters = 256;
    auto run = [&](const char* name, int S, int depth, int bps, int lanes, auto launch) {
        const int blocks = sms * bps;
        launch(blocks);
        cudaEventRecord(a);
        launch(blocks);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double accesses = (double)blocks * threads / lanes * iters;
        printf("{\"access\": \"%s\", \"bytes\": %d, \"in_flight\": %d, \"blocks_per_sm\": %d, \"ms\": %.3f, "
               "\"GBps\": %.1f, \"Gaccess_s\": %.2f}\n",
               name, S, depth, bps, ms, accesses * S / ms / 1e6, accesses / ms / 1e6);
    };
#define RUN(S, D, B)                                                                          \
    run(#S "B", S, D, B, S >= 16 ? S / 16 : 1, [&](int blocks) {                                                    \
        k_rand<S, D><<<blocks, threads>>>(buf, (uint32_t)(bytes / S), iters, sink); \
    });
    RUN(8, 4, 8)
    RUN(8, 8, 8)
    RUN(16, 4, 8)
    RUN(16, 8, 8)
    RUN(32, 4, 8)
    RUN(32, 8, 8)
    RUN(64, 4, 8)
    RUN(64, 8, 8)
    RUN(64, 16, 4)
    RUN(128, 4, 8)
    RUN(128, 8, 8)
    RUN(256, 4, 8)
    RUN(256, 8, 8)
#define RUNW(S, W)                                                                              \
    run(#S "B/w" #W, S, 4, 8, S / W, [&](int blocks) {                                                 \
        k_randw<S, W><<<blocks, threads>>>((const uint8_t*)buf, (uint32_t)(bytes / S), iters, sink); \
    });
    RUNW(32, 4)
    RUNW(32, 8)
    RUNW(32, 16)
    RUNW(64, 4)
    RUNW(64, 8)
    RUNW(64, 16)
    RUNW(128, 4)
    RUNW(128, 8)
    RUNW(128, 16)
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    return 0;
}

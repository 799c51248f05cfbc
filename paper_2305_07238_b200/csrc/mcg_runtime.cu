// Device runtime and C ABI: contexts, the HBM material cache, batched
// descriptor/codec/probe kernels, the probe microbenchmark, per-point VM
// execution and scene upload. Reference behaviour cited per entry point
// (paths relative to /root/reference/proj/core).
#include <cub/cub.cuh>

#include <algorithm>
#include <cstring>
#include <fstream>
#include <functional>
#include <limits>
#include <vector>

#include "host_scene.hpp"
#include "mcg_ctx.cuh"

using namespace mcg;
using mcgd::CacheView;

namespace mcg {

cudaEvent_t take_event(mcg_ctx* ctx) {
    if (!ctx->event_pool.empty()) {
        cudaEvent_t e = ctx->event_pool.back();
        ctx->event_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cuda_check(cudaEventCreate(&e), "cudaEventCreate");
    return e;
}

void resolve_events(mcg_ctx* ctx) {
    for (EventRec& r : ctx->pending) {
        cuda_check(cudaEventSynchronize(r.b), "cudaEventSynchronize");
        float ms = 0.0f;
        cudaEventElapsedTime(&ms, r.a, r.b);
        KernelAcc& acc = ctx->times[r.name];
        acc.launches += 1;
        acc.ms += ms;
        acc.bytes += r.bytes;
        ctx->event_pool.push_back(r.a);
        ctx->event_pool.push_back(r.b);
    }
    ctx->pending.clear();
}

void sort_pairs_u64(mcg_ctx* ctx, const unsigned long long* ki, unsigned long long* ko,
                    const unsigned long long* vi, unsigned long long* vo, size_t n, int end_bit) {
    size_t bytes = 0;
    cuda_check(cub::DeviceRadixSort::SortPairs(nullptr, bytes, ki, ko, vi, vo, static_cast<int>(n), 0,
                                               end_bit, ctx->stream),
               "cub sort (size)");
    ctx->cub_temp.ensure(std::max<size_t>(bytes, 256));
    cuda_check(cub::DeviceRadixSort::SortPairs(ctx->cub_temp.p, bytes, ki, ko, vi, vo,
                                               static_cast<int>(n), 0, end_bit, ctx->stream),
               "cub sort");
    ++ctx->library_sorts;  // CUB's kernels: library code, not counted in launches
}

void sort_pairs_u32(mcg_ctx* ctx, const uint32_t* ki, uint32_t* ko, const uint32_t* vi,
                    uint32_t* vo, size_t n, int end_bit, cudaStream_t stream, DevMem* temp) {
    const cudaStream_t st = stream ? stream : ctx->stream;
    DevMem& tmp = temp ? *temp : ctx->cub_temp;
    size_t bytes = 0;
    cuda_check(cub::DeviceRadixSort::SortPairs(nullptr, bytes, ki, ko, vi, vo, static_cast<int>(n), 0,
                                               end_bit, st),
               "cub sort (size)");
    tmp.ensure(std::max<size_t>(bytes, 256));
    cudaEvent_t a = nullptr;
    if (ctx->profile) {
        a = take_event(ctx);
        cudaEventRecord(a, st);
    }
    cuda_check(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, ki, ko, vi, vo,
                                               static_cast<int>(n), 0, end_bit, st),
               "cub sort");
    if (ctx->profile) {  // timed with the kernels, but CUB's launches are not counted as ours
        cudaEvent_t b = take_event(ctx);
        cudaEventRecord(b, st);
        ctx->pending.push_back({"sort (cub)", a, b, static_cast<double>(n) * 16.0 * ((end_bit + 7) / 8)});
    }
    ++ctx->library_sorts;
}

}  // namespace mcg

// ===========================================================================
// Kernels
// ===========================================================================
namespace {

using mcgd::Desc;

__device__ __forceinline__ Desc load_desc(const mcg_descriptor* d, size_t i) {
    // 20-byte records: five 32-bit words.
    const uint32_t* w = reinterpret_cast<const uint32_t*>(d) + 5 * i;
    return Desc{__ldg(w), __ldg(w + 1), __ldg(w + 3), __ldg(w + 4), __ldg(w + 2) & 0xffu};
}

__global__ void k_hash(const mcg_descriptor* d, size_t n, uint64_t* cell, uint32_t* check) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    uint64_t h;
    uint32_t c;
    mcgd::hash_desc(load_desc(d, i), h, c);
    cell[i] = h;
    check[i] = c;
}

__global__ void k_encode(const float* rgb, size_t n, uint32_t* out) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    out[i] = mcgd::encode_rgbe(rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]);
}

__global__ void k_decode(const uint32_t* in, size_t n, float* rgb) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const float3 c = mcgd::decode_rgbe(in[i]);
    rgb[3 * i] = c.x;
    rgb[3 * i + 1] = c.y;
    rgb[3 * i + 2] = c.z;
}

__global__ void k_mip_texel(const float* uv, const float* g1, const float* g2, size_t n, int off,
                            uint8_t* mip, uint32_t* txy) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const uint32_t m = mcgd::mip_level(g1[2 * i], g1[2 * i + 1], g2[2 * i], g2[2 * i + 1], off);
    mip[i] = static_cast<uint8_t>(m);
    txy[2 * i] = mcgd::texel_index(uv[2 * i], m);
    txy[2 * i + 1] = mcgd::texel_index(uv[2 * i + 1], m);
}

// Counters: [0] lookups [1] hits [2] inserts_won [3] inserts_lost_full [4] lost_race
__global__ void k_lookup(CacheView c, const mcg_descriptor* d, size_t n, uint8_t* hit, float* rgb,
                         unsigned long long* counters) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    const bool valid = i < n;
    uint64_t h = 0;
    uint32_t chk = 0;
    if (valid) mcgd::hash_desc(load_desc(d, i), h, chk);
    const uint64_t cell = valid ? mcgd::fast_mod(h, c.n_cells, c.magic) : 0;
    __shared__ ulonglong2 s_tile[8 * 4 * 32];   // blockDim 256: 4 rounds x 32 lanes per warp
    const mcgd::Probe p = mcgd::probe_lanes_smem(c, cell, chk, valid, s_tile + (threadIdx.x >> 5) * 128u);
    uint32_t hits = 0, looks = 0;
    if (valid) {
        looks = 1;
        hits = p.hit;
        if (hit) hit[i] = p.hit;
        if (rgb) {
            const float3 v = p.hit ? mcgd::decode_rgbe(p.payload) : make_float3(0.f, 0.f, 0.f);
            rgb[3 * i] = v.x;
            rgb[3 * i + 1] = v.y;
            rgb[3 * i + 2] = v.z;
        }
    }
    mcgd::warp_add(counters + 0, looks);
    mcgd::warp_add(counters + 1, hits);
}

// Concurrent update(): scan, then a single CAS from zero (cache.cpp:94-119).
__global__ void k_update(CacheView c, const mcg_descriptor* d, const float* rgb, size_t n,
                         uint8_t* outcome, uint64_t* slot_out, uint64_t* packed_out,
                         unsigned long long* counters) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    const bool valid = i < n;
    uint64_t h = 0;
    uint32_t chk = 0;
    const Desc dd = valid ? load_desc(d, i) : Desc{0u, 0u, 0u, 0u, 0u};
    if (valid) mcgd::hash_desc(dd, h, chk);
    const uint64_t cell = valid ? mcgd::fast_mod(h, c.n_cells, c.magic) : 0;
    const uint64_t base = cell * c.n_entries;   // logical slot index of the cell
    __shared__ ulonglong2 s_tile[8 * 4 * 32];   // blockDim 256: 4 rounds x 32 lanes per warp
    const mcgd::Probe p = mcgd::probe_lanes_smem(c, cell, chk, valid, s_tile + (threadIdx.x >> 5) * 128u);
    uint32_t won = 0, full = 0, lost = 0;
    if (valid) {
        int res;
        uint64_t slot = ~0ull, packed = 0;
        if (p.hit) {
            res = MCG_INSERT_ALREADY_PRESENT;
            slot = base + p.where;
            packed = (static_cast<uint64_t>(chk) << 32) | p.payload;
        } else {
            const uint32_t payload = mcgd::encode_rgbe(rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]);
            int32_t at = -1;
            res = mcgd::insert_at(c, cell, p.where, chk, payload, &at);
            if (res != MCG_INSERT_CELL_FULL) {
                slot = base + static_cast<uint32_t>(at);
                packed = (static_cast<uint64_t>(chk) << 32) | payload;
                if (res == MCG_INSERT_ALREADY_PRESENT) packed = *mcgd::slot_ptr(c, cell, static_cast<uint32_t>(at));
            }
            if (c.ilog && res == MCG_INSERT_WON) {
                mcgd::log_insert(c, dd.mat, dd.node, dd.mip, dd.tx, dd.ty, static_cast<uint32_t>(at), payload);
            }
        }
        won = res == MCG_INSERT_WON;
        full = res == MCG_INSERT_CELL_FULL;
        lost = res == MCG_INSERT_LOST_RACE;
        if (outcome) outcome[i] = static_cast<uint8_t>(res);
        if (slot_out) slot_out[i] = slot;
        if (packed_out) packed_out[i] = packed;
    }
    mcgd::warp_add(counters + 2, won);
    mcgd::warp_add(counters + 3, full);
    mcgd::warp_add(counters + 4, lost);
}

// Builds sortable records for an ordered batch: key = cell << ob | index.
__global__ void k_prepare_ordered(CacheView c, const mcg_descriptor* d, const float* rgb, size_t n,
                                  int ob, unsigned long long* keys, unsigned long long* vals) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    uint64_t h;
    uint32_t chk;
    mcgd::hash_desc(load_desc(d, i), h, chk);
    const uint64_t cell = mcgd::fast_mod(h, c.n_cells, c.magic);
    keys[i] = (cell << ob) | i;
    vals[i] = (static_cast<unsigned long long>(chk) << 32) |
              mcgd::encode_rgbe(rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]);
}

// One thread per cell segment of the sorted records applies them in order
// with update() semantics; a single writer per cell, so no atomics.
__global__ void k_apply_ordered(CacheView c, const unsigned long long* keys,
                                const unsigned long long* vals, size_t n, int ob, uint8_t* outcome,
                                uint64_t* slot_out, uint64_t* packed_out,
                                unsigned long long* counters) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    uint32_t won = 0, full = 0;
    if (i < n) {
        const uint64_t cell = keys[i] >> ob;
        if (i == 0 || (keys[i - 1] >> ob) != cell) {
            const unsigned long long omask = ob >= 64 ? ~0ull : ((1ull << ob) - 1ull);
            for (size_t j = i; j < n && (keys[j] >> ob) == cell; ++j) {
                const uint32_t chk = static_cast<uint32_t>(vals[j] >> 32);
                const unsigned long long packed = vals[j];
                int res = MCG_INSERT_CELL_FULL;
                uint64_t slot = ~0ull, pk = 0;
                for (uint32_t s = 0; s < c.n_entries; ++s) {
                    uint64_t* word = mcgd::slot_ptr(c, cell, s);
                    const uint64_t cur = *word;
                    if (static_cast<uint32_t>(cur >> 32) == chk) {
                        res = MCG_INSERT_ALREADY_PRESENT;
                        slot = cell * c.n_entries + s;
                        pk = cur;
                        break;
                    }
                    if (cur == 0ull) {
                        *word = packed;
                        res = MCG_INSERT_WON;
                        slot = cell * c.n_entries + s;
                        pk = packed;
                        break;
                    }
                }
                won += res == MCG_INSERT_WON;
                full += res == MCG_INSERT_CELL_FULL;
                const size_t idx = keys[j] & omask;
                if (outcome) outcome[idx] = static_cast<uint8_t>(res);
                if (slot_out) slot_out[idx] = slot;
                if (packed_out) packed_out[idx] = pk;
            }
        }
    }
    mcgd::warp_add(counters + 2, won);
    mcgd::warp_add(counters + 3, full);
}

__global__ void k_occupied(const uint64_t* slots, uint64_t n, unsigned long long* out) {
    uint32_t cnt = 0;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        cnt += slots[i] != 0ull;
    }
    mcgd::warp_add(out, cnt);
}

// Probe microbenchmark: descriptors are generated in registers
// (mat < 8, node < 256, mip <= 16, texels uniform in 2^mip) so the kernel's
// DRAM traffic is the table's alone.
// One splitmix64 output feeds every field (bits 0-2 mat, 3-10 node, 11-31 ->
// mip mod 17, 32-47 texel x, 48-63 texel y; mip <= 16 so 16 texel bits
// suffice), so the generator costs one mix64 next to the probe's six.
__device__ __forceinline__ Desc bench_desc(uint64_t seed, uint64_t i) {
    const uint64_t h = mcgd::mix64(seed + 0x9e3779b97f4a7c15ull * (i + 1));
    const uint32_t lo = static_cast<uint32_t>(h), hi = static_cast<uint32_t>(h >> 32);
    const uint32_t mip = (lo >> 11) % 17u;
    const uint32_t mask = (1u << mip) - 1u;
    return Desc{lo & 7u, (lo >> 3) & 255u, hi & mask, (hi >> 16) & mask, mip};
}

#ifndef MCG_PROBE_MINB
#define MCG_PROBE_MINB 1
#endif
template <int kVariant>
__global__ void __launch_bounds__(256, MCG_PROBE_MINB) k_probe_bench(CacheView c, uint64_t n, uint64_t seed,
                                                     int phase, unsigned long long* counters) {
    uint32_t looks = 0, hits = 0, won = 0, full = 0, inserts = 0;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    // Warp-uniform trip count (the cooperative variant needs every lane).
    for (uint64_t i0 = blockIdx.x * static_cast<uint64_t>(blockDim.x) + (threadIdx.x & ~31u); i0 < n;
         i0 += stride) {
        const uint64_t i = i0 + (threadIdx.x & 31u);
        const bool valid = i < n;
        uint64_t h;
        uint32_t chk;
        mcgd::hash_desc(bench_desc(seed, i), h, chk);
        const uint64_t cell = mcgd::fast_mod(h, c.n_cells, c.magic);
        mcgd::Probe p;
        if (kVariant == 4) p = mcgd::probe_warp16(c, cell, chk, valid);
        else if (kVariant == 2) p = mcgd::probe_warp<10>(c, cell, chk, valid);
        else if (kVariant == 1) p = valid ? mcgd::probe_cell_t<5>(c, cell, chk) : mcgd::Probe{0u, -1, false};
        else if (kVariant == 3) p = valid ? mcgd::probe_cell_blk(c, cell, chk) : mcgd::Probe{0u, -1, false};
        else p = valid ? mcgd::probe_cell_t<1>(c, cell, chk) : mcgd::Probe{0u, -1, false};
        if (!valid) continue;
        const bool insert = phase == 0 || (phase == 2 && (i & 1u));
        if (!insert) {
            ++looks;
            hits += p.hit;
        } else {
            ++inserts;
            if (!p.hit) {
                const int r = mcgd::insert_at(c, cell, p.where, chk,
                                              static_cast<uint32_t>(h) | 0x80000000u);
                won += r == MCG_INSERT_WON;
                full += r == MCG_INSERT_CELL_FULL;
            }
        }
    }
    mcgd::warp_add(counters + 0, looks);
    mcgd::warp_add(counters + 1, hits);
    mcgd::warp_add(counters + 2, won);
    mcgd::warp_add(counters + 3, full);
    mcgd::warp_add(counters + 5, inserts);
}

// Software-pipelined cooperative probe (variants 5/6): a warp takes U batches
// of 32 descriptors per step, issues every head load of all U batches (4U
// 16-byte loads per lane in flight), then hashes the next step's descriptors
// while the loads are outstanding, and only then resolves the scans. Same
// scan, same outcomes as variant 4; more DRAM requests in flight per warp
// and the hashing off the critical path.
// Register budgets: 64 (U = 1, 4 blocks of 256 per SM), 80 (U = 2, 3 blocks),
// 128 (U = 4, 2 blocks): more loads in flight per SM as U grows.
// kNoHash (diagnostic only, variants 8/9): the cell and check come from one
// multiply-high of a counter hash instead of the reference's descriptor hash,
// to measure what the hashing costs the probe.
template <int U, bool kNoHash = false, bool kSmem = false>
#ifndef MCG_PIPE1_MINB
#define MCG_PIPE1_MINB 4
#endif
#ifndef MCG_PIPE2_MINB
#define MCG_PIPE2_MINB 3
#endif
__global__ void __launch_bounds__(256, U == 1 ? MCG_PIPE1_MINB : (U == 2 ? MCG_PIPE2_MINB : 2)) k_probe_bench_pipe(CacheView c, uint64_t n, uint64_t seed,
                                                          int phase, unsigned long long* counters) {
    uint32_t looks = 0, hits = 0, won = 0, full = 0, inserts = 0;
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t step = static_cast<uint64_t>(gridDim.x) * blockDim.x * U;
    __shared__ ulonglong2 s_tile[kSmem ? 8 * 4 * 32 : 1];   // per warp: 4 rounds x 32 lanes
    ulonglong2* tile = s_tile + (kSmem ? (threadIdx.x >> 5) * 128u : 0u);
    uint64_t i0 = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + (threadIdx.x & ~31u)) * U;
    uint64_t cell[U], h[U];
    uint32_t chk[U];
    auto gen = [&](uint64_t i, uint64_t& hh, uint32_t& ck, uint64_t& cl) {
        if (kNoHash) {
            hh = (seed + i) * 0x9e3779b97f4a7c15ull;
            ck = static_cast<uint32_t>(hh) | 1u;
            cl = ((hh >> 32) * c.n_cells) >> 32;
        } else {
            mcgd::hash_desc(bench_desc(seed, i), hh, ck);
            cl = mcgd::fast_mod(hh, c.n_cells, c.magic);
        }
    };
#pragma unroll
    for (int u = 0; u < U; ++u) gen(i0 + 32u * u + lane, h[u], chk[u], cell[u]);
    for (; i0 < n; i0 += step) {
        ulonglong2 w[U][4];
#pragma unroll
        for (int u = 0; u < U; ++u) mcgd::probe_warp16_issue(c, cell[u], i0 + 32u * u + lane < n, w[u]);
        uint64_t ncell[U], nh[U];
        uint32_t nchk[U];
#pragma unroll
        for (int u = 0; u < U; ++u) gen(i0 + step + 32u * u + lane, nh[u], nchk[u], ncell[u]);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t i = i0 + 32u * u + lane;
            const bool valid = i < n;
            const mcgd::Probe p = kSmem ? mcgd::probe_warp16_resolve_smem(c, cell[u], chk[u], valid, w[u], tile)
                                        : mcgd::probe_warp16_resolve(c, cell[u], chk[u], valid, w[u]);
            if (valid) {
                const bool insert = phase == 0 || (phase == 2 && (i & 1u));
                if (!insert) {
                    ++looks;
                    hits += p.hit;
                } else {
                    ++inserts;
                    if (!p.hit) {
                        const int r = mcgd::insert_at(c, cell[u], p.where, chk[u],
                                                      static_cast<uint32_t>(h[u]) | 0x80000000u);
                        won += r == MCG_INSERT_WON;
                        full += r == MCG_INSERT_CELL_FULL;
                    }
                }
            }
            cell[u] = ncell[u];
            h[u] = nh[u];
            chk[u] = nchk[u];
        }
    }
    mcgd::warp_add(counters + 0, looks);
    mcgd::warp_add(counters + 1, hits);
    mcgd::warp_add(counters + 2, won);
    mcgd::warp_add(counters + 3, full);
    mcgd::warp_add(counters + 5, inserts);
}

// Replay of a recorded descriptor trace: in trace order, each
// warp takes 32 consecutive lookups, probes them cooperatively and inserts
// the misses (payload from the hash), as the VM's lookup + store would.
template <bool kPipe>
__global__ void __launch_bounds__(256, 4) k_probe_replay(CacheView c, const mcg_descriptor* d, uint64_t n,
                                                         unsigned long long* counters) {
    // kPipe: software-pipelined like k_probe_bench_pipe -- the step's head
    // loads are issued, then the next step's descriptors are read and hashed
    // while they are outstanding (one round trip for both). Off by default:
    // a render's trace is coherent and mostly hits L2, where it measured slower.
    uint32_t looks = 0, hits = 0, won = 0, full = 0;
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    __shared__ ulonglong2 s_tile[8 * 4 * 32];   // per warp: 4 rounds x 32 lanes (probe_warp16_resolve_smem)
    ulonglong2* tile = s_tile + (threadIdx.x >> 5) * 128u;
    uint64_t i0 = blockIdx.x * static_cast<uint64_t>(blockDim.x) + (threadIdx.x & ~31u);
    auto gen = [&](uint64_t i, uint64_t& h, uint32_t& chk, uint64_t& cell) {
        h = 0;
        chk = 0;
        if (i < n) mcgd::hash_desc(load_desc(d, i), h, chk);
        cell = i < n ? mcgd::fast_mod(h, c.n_cells, c.magic) : 0;
    };
    uint64_t h, cell;
    uint32_t chk;
    gen(i0 + lane, h, chk, cell);
    for (; i0 < n; i0 += stride) {
        const uint64_t i = i0 + lane;
        const bool valid = i < n;
        ulonglong2 w[4];
        const bool coop = (c.head_n & 1u) == 0u && c.head_n >= 2u && c.head_n <= 8u;
        if (coop) mcgd::probe_warp16_issue(c, cell, valid, w);
        uint64_t nh = 0, ncell = 0;
        uint32_t nchk = 0;
        if (kPipe) gen(i + stride, nh, nchk, ncell);
        const mcgd::Probe p = coop ? mcgd::probe_warp16_resolve_smem(c, cell, chk, valid, w, tile)
                                   : (valid ? mcgd::probe_cell(c, cell, chk) : mcgd::Probe{0u, -1, false});
        if (valid) {
            ++looks;
            hits += p.hit;
            if (!p.hit) {
                const int r = mcgd::insert_at(c, cell, p.where, chk, static_cast<uint32_t>(h) | 0x80000000u);
                won += r == MCG_INSERT_WON;
                full += r == MCG_INSERT_CELL_FULL;
            }
        }
        if (kPipe) {
            h = nh;
            chk = nchk;
            cell = ncell;
        } else {
            gen(i + stride, h, chk, cell);
        }
    }
    mcgd::warp_add(counters + 0, looks);
    mcgd::warp_add(counters + 1, hits);
    mcgd::warp_add(counters + 2, won);
    mcgd::warp_add(counters + 3, full);
}

// Per-point VM execution for mcg_execute_batch: every lane runs the same slot.
template <bool kDeferred>
__global__ void k_execute(mcgd::SceneView S, CacheView C, int cache_on, int mip_offset,
                          uint32_t slot, const float* sp, size_t n, int max_stack, float* values,
                          uint32_t* nodes, uint32_t* instrs, mcgd::StoreQueue q,
                          unsigned long long* counters) {
    extern __shared__ float smem[];
    __shared__ uint8_t s_perm[256];
    mcgd::stage_perm(s_perm);
    __syncthreads();
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    const bool valid = i < n;
    const unsigned grp = __ballot_sync(mcgd::kFull, valid);
    if (!valid) return;
    mcgd::Stack st{smem, smem + max_stack * blockDim.x, smem + 2 * max_stack * blockDim.x,
                   static_cast<int>(blockDim.x), static_cast<int>(threadIdx.x), max_stack};
    const float* p = sp + 15 * i;
    const mcgd::ShadeIn in{p[0], p[1], p[2], p[3], p[4], p[5], p[6], p[7], p[8],
                           p[9], p[10], p[11], p[12], p[13], p[14]};
    mcgd::VmCounters cnt;
    const mcgd::VmResult r = mcgd::run_program<kDeferred>(
        S, C, cache_on != 0, mip_offset, slot, in, grp, st, s_perm,
        static_cast<uint32_t>(i) << 6, q, cnt);
    values[4 * i] = r.value.x;
    values[4 * i + 1] = r.scalar ? r.value.x : r.value.y;
    values[4 * i + 2] = r.scalar ? r.value.x : r.value.z;
    values[4 * i + 3] = __uint_as_float(r.scalar ? 1u : 0u);
    nodes[i] = cnt.hits;
    instrs[i] = cnt.instrs;
    mcgd::warp_add(counters + 0, cnt.lookups);
    mcgd::warp_add(counters + 1, cnt.hits);
    mcgd::warp_add(counters + 2, cnt.won);
    mcgd::warp_add(counters + 3, cnt.full);
}

}  // namespace

namespace mcg {

void apply_ordered(mcg_ctx* ctx, mcg_cache* cache, const unsigned long long* keys,
                   const unsigned long long* vals, size_t n, int order_bits, uint8_t* d_outcome,
                   uint64_t* d_slot, uint64_t* d_packed, unsigned long long* d_stats) {
    if (n == 0) return;
    LaunchScope ls(ctx, "apply_ordered", static_cast<double>(n) * 16.0);
    k_apply_ordered<<<grid_for(n, 256), 256, 0, ctx->stream>>>(cache->view(), keys, vals, n,
                                                                order_bits, d_outcome, d_slot,
                                                                d_packed, d_stats);
    ls.done();
}

}  // namespace mcg

// ===========================================================================
// C ABI
// ===========================================================================
namespace {

template <typename T>
T* dev_upload(mcg_ctx* ctx, DevMem& m, const T* host, size_t n) {
    m.ensure(std::max<size_t>(n * sizeof(T), 16));
    if (n) cuda_check(cudaMemcpyAsync(m.p, host, n * sizeof(T), cudaMemcpyHostToDevice, ctx->stream), "H2D");
    return m.as<T>();
}

template <typename T>
void dev_download(mcg_ctx* ctx, T* host, const void* dev, size_t n) {
    if (n && host) cuda_check(cudaMemcpyAsync(host, dev, n * sizeof(T), cudaMemcpyDeviceToHost, ctx->stream), "D2H");
}

void need(bool ok, const char* msg) {
    if (!ok) fail(MCG_ERR_INVALID_ARGUMENT, msg);
}

void sync(mcg_ctx* ctx) { cuda_check(cudaStreamSynchronize(ctx->stream), "cudaStreamSynchronize"); }

}  // namespace

// Binned-SAH hierarchy over the reference BVH's leaves, collapsed to
// `width`-wide nodes in the entry layout of `quads` (entries: leaf
// (~first, count) with the leaf's own box, or node (index, -1) with the union
// of its leaves' boxes; unused entries zero). A node opens its largest-area
// internal entries until it holds `width` entries.
static std::vector<mcg_bvh_node> build_shadow_tree(const mcg_flat_scene& f, int width, int32_t& root_a,
                                                   int32_t& root_b) {
    const mcg_bvh_node* nodes = static_cast<const mcg_bvh_node*>(f.nodes);
    std::vector<mcg_bvh_node> leaves;
    for (uint32_t i = 0; i < f.n_nodes; ++i)
        if (nodes[i].a < 0) leaves.push_back(nodes[i]);
    std::vector<mcg_bvh_node> out;
    root_a = 0;
    root_b = 0;
    if (leaves.empty()) return out;
    if (leaves.size() == 1) {
        root_a = leaves[0].a;
        root_b = leaves[0].b;
        return out;
    }
    struct BNode { float lo[3], hi[3]; int32_t l = -1, r = -1, leaf = -1; };
    std::vector<BNode> bn;
    std::vector<int32_t> idx(leaves.size());
    for (size_t i = 0; i < idx.size(); ++i) idx[i] = static_cast<int32_t>(i);
    auto cen = [&](int32_t i, int a) { return 0.5f * (leaves[i].lo[a] + leaves[i].hi[a]); };
    auto area = [](const float* lo, const float* hi) {
        const float dx = hi[0] - lo[0], dy = hi[1] - lo[1], dz = hi[2] - lo[2];
        return dx * dy + dy * dz + dz * dx;
    };
    constexpr int kBins = 32;
    std::function<int32_t(size_t, size_t)> build = [&](size_t first, size_t count) -> int32_t {
        const int32_t id = static_cast<int32_t>(bn.size());
        bn.emplace_back();
        BNode nd;
        for (int a = 0; a < 3; ++a) {
            nd.lo[a] = std::numeric_limits<float>::infinity();
            nd.hi[a] = -std::numeric_limits<float>::infinity();
        }
        float clo[3], chi[3];
        for (int a = 0; a < 3; ++a) {
            clo[a] = std::numeric_limits<float>::infinity();
            chi[a] = -std::numeric_limits<float>::infinity();
        }
        for (size_t k = first; k < first + count; ++k) {
            const mcg_bvh_node& L = leaves[idx[k]];
            for (int a = 0; a < 3; ++a) {
                nd.lo[a] = std::min(nd.lo[a], L.lo[a]);
                nd.hi[a] = std::max(nd.hi[a], L.hi[a]);
                clo[a] = std::min(clo[a], cen(idx[k], a));
                chi[a] = std::max(chi[a], cen(idx[k], a));
            }
        }
        if (count == 1) {
            nd.leaf = idx[first];
            bn[id] = nd;
            return id;
        }
        // Binned SAH over centroids; fall back to an index median split.
        double best = std::numeric_limits<double>::infinity();
        int best_axis = -1, best_bin = 0;
        for (int a = 0; a < 3; ++a) {
            const float ext = chi[a] - clo[a];
            if (!(ext > 0.0f)) continue;
            int cnt[kBins] = {};
            float blo[kBins][3], bhi[kBins][3];
            for (int b = 0; b < kBins; ++b)
                for (int c = 0; c < 3; ++c) {
                    blo[b][c] = std::numeric_limits<float>::infinity();
                    bhi[b][c] = -std::numeric_limits<float>::infinity();
                }
            for (size_t k = first; k < first + count; ++k) {
                int b = static_cast<int>((cen(idx[k], a) - clo[a]) / ext * kBins);
                b = std::min(std::max(b, 0), kBins - 1);
                ++cnt[b];
                const mcg_bvh_node& L = leaves[idx[k]];
                for (int c = 0; c < 3; ++c) {
                    blo[b][c] = std::min(blo[b][c], L.lo[c]);
                    bhi[b][c] = std::max(bhi[b][c], L.hi[c]);
                }
            }
            // prefix/suffix sweeps
            float rlo[kBins][3], rhi[kBins][3];
            int rcnt[kBins];
            float alo[3], ahi[3];
            int acnt = 0;
            for (int c = 0; c < 3; ++c) {
                alo[c] = std::numeric_limits<float>::infinity();
                ahi[c] = -std::numeric_limits<float>::infinity();
            }
            for (int b = kBins - 1; b >= 0; --b) {
                acnt += cnt[b];
                for (int c = 0; c < 3; ++c) {
                    alo[c] = std::min(alo[c], blo[b][c]);
                    ahi[c] = std::max(ahi[c], bhi[b][c]);
                    rlo[b][c] = alo[c];
                    rhi[b][c] = ahi[c];
                }
                rcnt[b] = acnt;
            }
            for (int c = 0; c < 3; ++c) {
                alo[c] = std::numeric_limits<float>::infinity();
                ahi[c] = -std::numeric_limits<float>::infinity();
            }
            acnt = 0;
            for (int b = 0; b < kBins - 1; ++b) {
                acnt += cnt[b];
                for (int c = 0; c < 3; ++c) {
                    alo[c] = std::min(alo[c], blo[b][c]);
                    ahi[c] = std::max(ahi[c], bhi[b][c]);
                }
                if (acnt == 0 || rcnt[b + 1] == 0) continue;
                const double cost = static_cast<double>(area(alo, ahi)) * acnt +
                                    static_cast<double>(area(rlo[b + 1], rhi[b + 1])) * rcnt[b + 1];
                if (cost < best) {
                    best = cost;
                    best_axis = a;
                    best_bin = b;
                }
            }
        }
        size_t mid;
        if (best_axis < 0) {
            mid = first + count / 2;
        } else {
            const int a = best_axis;
            const float ext = chi[a] - clo[a];
            auto it = std::partition(idx.begin() + first, idx.begin() + first + count, [&](int32_t i) {
                int b = static_cast<int>((cen(i, a) - clo[a]) / ext * kBins);
                b = std::min(std::max(b, 0), kBins - 1);
                return b <= best_bin;
            });
            mid = static_cast<size_t>(it - idx.begin());
            if (mid == first || mid == first + count) mid = first + count / 2;
        }
        const int32_t l = build(first, mid - first);
        const int32_t r = build(mid, first + count - mid);
        nd.l = l;
        nd.r = r;
        bn[id] = nd;
        return id;
    };
    const int32_t root = build(0, leaves.size());
    std::function<int32_t(int32_t)> collapse = [&](int32_t x) -> int32_t {
        const int32_t q = static_cast<int32_t>(out.size() / width);
        out.resize(out.size() + width, mcg_bvh_node{{0, 0, 0}, 0, {0, 0, 0}, 0});
        std::vector<int32_t> entries{bn[x].l, bn[x].r};
        for (;;) {
            if (static_cast<int>(entries.size()) >= width) break;
            int best = -1;
            float best_area = -1.0f;
            for (size_t e = 0; e < entries.size(); ++e) {
                const BNode& b = bn[entries[e]];
                if (b.leaf >= 0) continue;
                const float a = area(b.lo, b.hi);
                if (a > best_area) {
                    best_area = a;
                    best = static_cast<int>(e);
                }
            }
            if (best < 0) break;
            const int32_t x2 = entries[best];
            entries[best] = bn[x2].l;
            entries.insert(entries.begin() + best + 1, bn[x2].r);
        }
        int k = 0;
        for (int32_t e : entries) {
            mcg_bvh_node rec;
            if (bn[e].leaf >= 0) {
                rec = leaves[bn[e].leaf];
            } else {
                std::memcpy(rec.lo, bn[e].lo, sizeof(rec.lo));
                std::memcpy(rec.hi, bn[e].hi, sizeof(rec.hi));
                rec.a = collapse(e);
                rec.b = -1;
            }
            out[static_cast<size_t>(width) * q + k++] = rec;
        }
        return q;
    };
    collapse(root);
    root_a = 0;
    root_b = -1;
    return out;
}

extern "C" {

mcg_status mcg_device_count(int32_t* count) {
    return guarded([&] {
        need(count != nullptr, "null out");
        int n = 0;
        cuda_check(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
        if (n == 0) fail(MCG_ERR_NO_DEVICE, "no CUDA device");
        *count = n;
    });
}

mcg_status mcg_create(const mcg_options* opt, mcg_ctx** out) {
    return guarded([&] {
        need(out != nullptr, "null out");
        int count = 0;
        cuda_check(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
        if (count == 0) fail(MCG_ERR_NO_DEVICE, "no CUDA device");
        const int n_dev = opt && opt->n_devices > 1 ? opt->n_devices : 1;
        std::vector<int> devs(n_dev);
        for (int k = 0; k < n_dev; ++k) {
            devs[k] = (opt && opt->devices) ? opt->devices[k] : (opt ? opt->device : 0) + k;
            need(devs[k] >= 0 && devs[k] < count, "device ordinal out of range");
        }
        need(n_dev == 1 || !(opt && opt->stream), "a multi-device context creates its own streams");
        const int dev = devs[0];
        cuda_check(cudaSetDevice(dev), "cudaSetDevice");
        auto* ctx = new mcg_ctx;
        ctx->device = dev;
        ctx->profile = opt && opt->profile;
        if (opt && opt->stream) {
            ctx->stream = static_cast<cudaStream_t>(opt->stream);
        } else {
            cudaError_t e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
            if (e != cudaSuccess) {
                delete ctx;
                cuda_check(e, "cudaStreamCreate");
            }
            ctx->own_stream = true;
        }
        ctx->stats_mem.ensure(4096);
        for (int k = 1; k < n_dev; ++k) {
            mcg_options po{devs[k], opt->profile, nullptr, 0, nullptr};
            mcg_ctx* peer = nullptr;
            const mcg_status st = mcg_create(&po, &peer);
            if (st != MCG_OK) {
                const std::string msg = mcg_last_error();
                mcg_destroy(ctx);
                fail(st, msg);
            }
            ctx->peers.push_back(peer);
            for (int j = 0; j < k; ++j) ctx->devices_distinct = ctx->devices_distinct && devs[j] != devs[k];
        }
        cuda_check(cudaSetDevice(dev), "cudaSetDevice");
        *out = ctx;
    });
}

mcg_status mcg_destroy(mcg_ctx* ctx) {
    if (!ctx) return MCG_OK;
    mcg::nccl_destroy(ctx);
    for (mcg_ctx* p : ctx->peers) mcg_destroy(p);
    ctx->peers.clear();
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    if (ctx->own_cache) mcg_cache_destroy(ctx->own_cache);
    ctx->scene.clear();
    for (DevMem* m : {&ctx->cub_temp, &ctx->scratch_a, &ctx->scratch_b, &ctx->scratch_c,
                      &ctx->scratch_d, &ctx->scratch_e, &ctx->path_mem, &ctx->queue_mem,
                      &ctx->stats_mem, &ctx->pix_mem}) {
        m->release();
    }
    for (int l = 0; l < mcg_ctx::kMaxLanes; ++l) {
        ctx->lane_cub[l].release();
        ctx->lane_path[l].release();
    }
    for (auto& r : ctx->pending) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    for (cudaEvent_t e : ctx->event_pool) cudaEventDestroy(e);
    if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
    if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
    if (ctx->aux) cudaStreamDestroy(ctx->aux);
    for (int l = 0; l < mcg_ctx::kMaxLanes; ++l) {
        if (ctx->lane_fork[l]) cudaEventDestroy(ctx->lane_fork[l]);
        if (ctx->lane_join[l]) cudaEventDestroy(ctx->lane_join[l]);
        if (ctx->lane_aux[l]) cudaStreamDestroy(ctx->lane_aux[l]);
        if (ctx->lane_stream[l]) cudaStreamDestroy(ctx->lane_stream[l]);
    }
    for (cudaEvent_t e : ctx->ev_lane) if (e) cudaEventDestroy(e);
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
    return MCG_OK;
}

mcg_status mcg_synchronize(mcg_ctx* ctx) {
    return guarded([&] {
        need(ctx != nullptr, "null ctx");
        sync(ctx);
        resolve_events(ctx);
    });
}

void* mcg_stream(mcg_ctx* ctx) { return ctx ? ctx->stream : nullptr; }

mcg_status mcg_kernel_times(mcg_ctx* ctx, mcg_kernel_time* out, int32_t cap, int32_t* n_out) {
    return guarded([&] {
        need(ctx != nullptr, "null ctx");
        sync(ctx);
        resolve_events(ctx);
        int32_t k = 0;
        for (const auto& [name, acc] : ctx->times) {
            if (out && k < cap) {
                std::memset(&out[k], 0, sizeof(mcg_kernel_time));
                std::snprintf(out[k].name, sizeof(out[k].name), "%s", name.c_str());
                out[k].launches = acc.launches;
                out[k].ms = acc.ms;
                out[k].algorithmic_bytes = acc.bytes;
            }
            ++k;
        }
        if (n_out) *n_out = k;
    });
}

mcg_status mcg_kernel_times_reset(mcg_ctx* ctx) {
    return guarded([&] {
        need(ctx != nullptr, "null ctx");
        sync(ctx);
        resolve_events(ctx);
        ctx->times.clear();
        ctx->launches = 0;
    });
}

uint64_t mcg_launch_count(mcg_ctx* ctx) { return ctx ? ctx->launches : 0; }

mcg_status mcg_hash_batch(mcg_ctx* ctx, const mcg_descriptor* d, size_t n, uint64_t* cell_hash,
                          uint32_t* check) {
    return guarded([&] {
        need(ctx && d && cell_hash && check, "null argument");
        if (!n) return;
        auto* dd = dev_upload(ctx, ctx->scratch_a, d, n);
        ctx->scratch_b.ensure(n * 8);
        ctx->scratch_c.ensure(n * 4);
        LaunchScope ls(ctx, "hash", n * 20.0 + n * 12.0);
        k_hash<<<grid_for(n, 256), 256, 0, ctx->stream>>>(dd, n, ctx->scratch_b.as<uint64_t>(),
                                                         ctx->scratch_c.as<uint32_t>());
        ls.done();
        dev_download(ctx, cell_hash, ctx->scratch_b.p, n);
        dev_download(ctx, check, ctx->scratch_c.p, n);
        sync(ctx);
    });
}

mcg_status mcg_encode_batch(mcg_ctx* ctx, const float* rgb, size_t n, uint32_t* packed) {
    return guarded([&] {
        need(ctx && rgb && packed, "null argument");
        if (!n) return;
        auto* d = dev_upload(ctx, ctx->scratch_a, rgb, 3 * n);
        ctx->scratch_b.ensure(n * 4);
        LaunchScope ls(ctx, "encode", n * 16.0);
        k_encode<<<grid_for(n, 256), 256, 0, ctx->stream>>>(d, n, ctx->scratch_b.as<uint32_t>());
        ls.done();
        dev_download(ctx, packed, ctx->scratch_b.p, n);
        sync(ctx);
    });
}

mcg_status mcg_decode_batch(mcg_ctx* ctx, const uint32_t* packed, size_t n, float* rgb) {
    return guarded([&] {
        need(ctx && rgb && packed, "null argument");
        if (!n) return;
        auto* d = dev_upload(ctx, ctx->scratch_a, packed, n);
        ctx->scratch_b.ensure(n * 12);
        LaunchScope ls(ctx, "decode", n * 16.0);
        k_decode<<<grid_for(n, 256), 256, 0, ctx->stream>>>(d, n, ctx->scratch_b.as<float>());
        ls.done();
        dev_download(ctx, rgb, ctx->scratch_b.p, 3 * n);
        sync(ctx);
    });
}

mcg_status mcg_mip_texel_batch(mcg_ctx* ctx, const float* uv, const float* g1, const float* g2,
                               size_t n, int32_t mip_offset, uint8_t* mip, uint32_t* texel_xy) {
    return guarded([&] {
        need(ctx && uv && g1 && g2 && mip && texel_xy, "null argument");
        if (!n) return;
        auto* duv = dev_upload(ctx, ctx->scratch_a, uv, 2 * n);
        auto* dg1 = dev_upload(ctx, ctx->scratch_b, g1, 2 * n);
        auto* dg2 = dev_upload(ctx, ctx->scratch_c, g2, 2 * n);
        ctx->scratch_d.ensure(n);
        ctx->scratch_e.ensure(n * 8);
        LaunchScope ls(ctx, "mip_texel", n * 33.0);
        k_mip_texel<<<grid_for(n, 256), 256, 0, ctx->stream>>>(duv, dg1, dg2, n, mip_offset,
                                                              ctx->scratch_d.as<uint8_t>(),
                                                              ctx->scratch_e.as<uint32_t>());
        ls.done();
        dev_download(ctx, mip, ctx->scratch_d.p, n);
        dev_download(ctx, texel_xy, ctx->scratch_e.p, 2 * n);
        sync(ctx);
    });
}

// ---- cache -----------------------------------------------------------------

mcg_status mcg_cache_create(mcg_ctx* ctx, uint64_t n_cells, uint32_t n_entries, mcg_cache** out) {
    return guarded([&] {
        need(ctx && out, "null argument");
        if (n_cells == 0 || n_entries == 0) {
            fail(MCG_ERR_INVALID_ARGUMENT, "cache dimensions must be nonzero");
        }
        uint64_t bytes = 0;
        const mcg_status s = mcg_memory_bytes(n_cells, n_entries, &bytes);
        if (s != MCG_OK) fail(s, mcg_last_error());
        if (n_cells >= (1ull << 32)) fail(MCG_ERR_INVALID_ARGUMENT, "n_cells must be < 2^32");
        auto* c = new mcg_cache;
        c->ctx = ctx;
        c->n_cells = n_cells;
        c->n_entries = n_entries;
        c->head_n = head_slots(n_entries);
        c->magic = mod_magic(n_cells);
        c->local_cells = n_cells;
        cudaError_t e = cudaMalloc(&c->slots, bytes);
        if (e == cudaSuccess) e = cudaMalloc(&c->counters, 8 * sizeof(unsigned long long));
        if (e != cudaSuccess) {
            if (c->slots) cudaFree(c->slots);
            delete c;
            cuda_check(e, "cudaMalloc(cache)");
        }
        cuda_check(cudaMemsetAsync(c->slots, 0, bytes, ctx->stream), "memset cache");
        cuda_check(cudaMemsetAsync(c->counters, 0, 8 * sizeof(unsigned long long), ctx->stream), "memset");
        sync(ctx);
        *out = c;
    });
}

// Logical slots [first, first + n) of this object's cells (cell-major,
// n_entries per cell: the reference's dump order) from the head/tail arrays.
static void read_logical(mcg_cache* cache, uint64_t first, size_t n, uint64_t* out) {
    mcg_ctx* ctx = cache->ctx;
    const uint32_t ne = cache->n_entries, hn = cache->head_n, tn = ne - hn;
    if (tn == 0) {
        dev_download(ctx, out, cache->slots + first, n);
        sync(ctx);
        return;
    }
    const uint64_t c0 = first / ne, c1 = (first + n + ne - 1) / ne;
    std::vector<uint64_t> tmp((c1 - c0) * ne);
    // heads into columns [0, hn), tails into [hn, ne) of each logical cell
    cuda_check(cudaMemcpy2DAsync(tmp.data(), ne * 8ull, cache->slots + c0 * hn, hn * 8ull, hn * 8ull, c1 - c0,
                                 cudaMemcpyDeviceToHost, ctx->stream), "D2H heads");
    cuda_check(cudaMemcpy2DAsync(tmp.data() + hn, ne * 8ull, cache->tail() + c0 * tn, tn * 8ull, tn * 8ull,
                                 c1 - c0, cudaMemcpyDeviceToHost, ctx->stream), "D2H tails");
    sync(ctx);
    std::memcpy(out, tmp.data() + (first - c0 * ne), n * 8);
}

// The inverse: host words -> logical slots [first, first + n). Partial cells
// at either end are read first so their other words are kept.
static void write_logical(mcg_cache* cache, uint64_t first, size_t n, const uint64_t* in) {
    mcg_ctx* ctx = cache->ctx;
    const uint32_t ne = cache->n_entries, hn = cache->head_n, tn = ne - hn;
    if (tn == 0) {
        cuda_check(cudaMemcpyAsync(cache->slots + first, in, n * 8ull, cudaMemcpyHostToDevice, ctx->stream), "H2D");
        sync(ctx);
        return;
    }
    const uint64_t c0 = first / ne, c1 = (first + n + ne - 1) / ne;
    std::vector<uint64_t> tmp((c1 - c0) * ne);
    if (first % ne != 0 || (first + n) % ne != 0) read_logical(cache, c0 * ne, tmp.size(), tmp.data());
    std::memcpy(tmp.data() + (first - c0 * ne), in, n * 8);
    cuda_check(cudaMemcpy2DAsync(cache->slots + c0 * hn, hn * 8ull, tmp.data(), ne * 8ull, hn * 8ull, c1 - c0,
                                 cudaMemcpyHostToDevice, ctx->stream), "H2D heads");
    cuda_check(cudaMemcpy2DAsync(cache->tail() + c0 * tn, tn * 8ull, tmp.data() + hn, ne * 8ull, tn * 8ull,
                                 c1 - c0, cudaMemcpyHostToDevice, ctx->stream), "H2D tails");
    sync(ctx);
}

mcg_status mcg_cache_destroy(mcg_cache* cache) {
    if (!cache) return MCG_OK;
    cudaStreamSynchronize(cache->ctx->stream);
    for (void* p : cache->ipc_opened) cudaIpcCloseMemHandle(p);
    if (cache->trace) cudaFree(cache->trace);
    if (cache->trace_count) cudaFree(cache->trace_count);
    if (cache->ilog) cudaFree(cache->ilog);
    if (cache->ilog_count) cudaFree(cache->ilog_count);
    if (cache->stripes) cudaFree(cache->stripes);
    cudaFree(cache->slots);
    cudaFree(cache->counters);
    delete cache;
    return MCG_OK;
}

// ---- striped shared table --------------------------------------

mcg_status mcg_cache_create_stripe(mcg_ctx* ctx, uint64_t n_cells, uint32_t n_entries, uint32_t rank,
                                   uint32_t world, mcg_cache** out) {
    return guarded([&] {
        need(ctx && out, "null argument");
        need(world >= 1 && rank < world, "rank must be < world");
        if (n_cells == 0 || n_entries == 0) fail(MCG_ERR_INVALID_ARGUMENT, "cache dimensions must be nonzero");
        uint64_t bytes = 0;
        const mcg_status s = mcg_memory_bytes(n_cells, n_entries, &bytes);
        if (s != MCG_OK) fail(s, mcg_last_error());
        if (n_cells >= (1ull << 32)) fail(MCG_ERR_INVALID_ARGUMENT, "n_cells must be < 2^32");
        auto* c = new mcg_cache;
        c->ctx = ctx;
        c->n_cells = n_cells;
        c->n_entries = n_entries;
        c->magic = mod_magic(n_cells);
        c->world = world;
        c->rank = rank;
        c->head_n = head_slots(n_entries);
        c->local_cells = n_cells > rank ? (n_cells - rank + world - 1) / world : 0;
        const size_t local_bytes = std::max<uint64_t>(8, c->local_words() * 8);
        cudaError_t e = cudaMalloc(&c->slots, local_bytes);
        if (e == cudaSuccess) e = cudaMalloc(&c->counters, 8 * sizeof(unsigned long long));
        if (e != cudaSuccess) {
            if (c->slots) cudaFree(c->slots);
            delete c;
            cuda_check(e, "cudaMalloc(cache stripe)");
        }
        cuda_check(cudaMemsetAsync(c->slots, 0, local_bytes, ctx->stream), "memset stripe");
        cuda_check(cudaMemsetAsync(c->counters, 0, 8 * sizeof(unsigned long long), ctx->stream), "memset");
        sync(ctx);
        *out = c;
    });
}

static void upload_stripes(mcg_cache* c, const std::vector<uint64_t*>& ptrs) {
    if (!c->stripes) cuda_check(cudaMalloc(&c->stripes, ptrs.size() * sizeof(uint64_t*)), "cudaMalloc(stripes)");
    cuda_check(cudaMemcpyAsync(c->stripes, ptrs.data(), ptrs.size() * sizeof(uint64_t*), cudaMemcpyHostToDevice,
                               c->ctx->stream), "H2D stripes");
    sync(c->ctx);
}

mcg_status mcg_cache_attach_local(mcg_cache* cache, mcg_cache* const* stripes, uint32_t world) {
    return guarded([&] {
        need(cache && stripes, "null argument");
        need(world == cache->world, "world does not match the stripe's");
        std::vector<uint64_t*> ptrs(2 * world);
        for (uint32_t r = 0; r < world; ++r) {
            need(stripes[r] && stripes[r]->world == world && stripes[r]->rank == r &&
                     stripes[r]->n_cells == cache->n_cells && stripes[r]->n_entries == cache->n_entries,
                 "stripe r must be rank r of the same logical table");
            ptrs[2 * r] = stripes[r]->slots;
            ptrs[2 * r + 1] = stripes[r]->tail();
        }
        upload_stripes(cache, ptrs);
    });
}

mcg_status mcg_cache_ipc_handle(mcg_cache* cache, void* out, size_t cap) {
    return guarded([&] {
        need(cache && out, "null argument");
        need(cap >= sizeof(cudaIpcMemHandle_t), "handle buffer too small (64 bytes)");
        cudaIpcMemHandle_t h;
        cuda_check(cudaIpcGetMemHandle(&h, cache->slots), "cudaIpcGetMemHandle");
        std::memcpy(out, &h, sizeof(h));
    });
}

mcg_status mcg_cache_attach_ipc(mcg_cache* cache, const void* handles, uint32_t world) {
    return guarded([&] {
        need(cache && handles, "null argument");
        need(world == cache->world, "world does not match the stripe's");
        need(cache->ipc_opened.empty(), "stripes already attached");
        std::vector<uint64_t*> ptrs(2 * world);
        const auto* hb = static_cast<const unsigned char*>(handles);
        for (uint32_t r = 0; r < world; ++r) {
            // stripe r's cells and the offset of its tail array
            const uint64_t cells_r = cache->n_cells > r ? (cache->n_cells - r + world - 1) / world : 0;
            if (r == cache->rank) {
                ptrs[2 * r] = cache->slots;
                ptrs[2 * r + 1] = cache->tail();
                continue;
            }
            cudaIpcMemHandle_t h;
            std::memcpy(&h, hb + static_cast<size_t>(r) * sizeof(h), sizeof(h));
            void* p = nullptr;
            cuda_check(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
            cache->ipc_opened.push_back(p);
            ptrs[2 * r] = static_cast<uint64_t*>(p);
            ptrs[2 * r + 1] = cache->n_entries > cache->head_n ? ptrs[2 * r] + cells_r * cache->head_n : nullptr;
        }
        upload_stripes(cache, ptrs);
    });
}

mcg_status mcg_cache_stripe_info(const mcg_cache* cache, uint32_t* rank, uint32_t* world,
                                 uint64_t* local_cells) {
    return guarded([&] {
        need(cache != nullptr, "null cache");
        if (rank) *rank = cache->rank;
        if (world) *world = cache->world;
        if (local_cells) *local_cells = cache->local_cells;
    });
}

mcg_status mcg_cache_clear(mcg_cache* cache) {
    return guarded([&] {
        need(cache != nullptr, "null cache");
        cuda_check(cudaMemsetAsync(cache->slots, 0, cache->local_words() * 8,
                                   cache->ctx->stream), "memset cache");
        cuda_check(cudaMemsetAsync(cache->counters, 0, 8 * sizeof(unsigned long long),
                                   cache->ctx->stream), "memset counters");
    });
}

mcg_status mcg_cache_shape(const mcg_cache* cache, uint64_t* n_cells, uint32_t* n_entries) {
    return guarded([&] {
        need(cache != nullptr, "null cache");
        if (n_cells) *n_cells = cache->n_cells;
        if (n_entries) *n_entries = cache->n_entries;
    });
}

uint64_t* mcg_cache_device_slots(mcg_cache* cache) { return cache ? cache->slots : nullptr; }

static void update_device(mcg_cache* cache, const mcg_descriptor* dd, const float* drgb, size_t n,
                          int32_t mode, uint8_t* d_out, uint64_t* d_slot, uint64_t* d_packed) {
    mcg_ctx* ctx = cache->ctx;
    if (!n) return;
    need(cache->world == 1 || cache->stripes, "striped table: attach the stripes first");
    if (mode == MCG_APPLY_CONCURRENT) {
        LaunchScope ls(ctx, "cache_update", n * (8.0 * cache->n_entries));
        k_update<<<grid_for(n, 256), 256, 0, ctx->stream>>>(cache->view(), dd, drgb, n, d_out,
                                                           d_slot, d_packed, cache->counters);
        ls.done();
        return;
    }
    need(mode == MCG_APPLY_ORDERED, "unknown apply mode");
    const int ob = std::max(1, bits_for(n - 1));
    const int end_bit = ob + bits_for(cache->n_cells - 1);
    need(end_bit <= 64, "ordered batch too large for 64-bit keys");
    ctx->queue_mem.ensure(n * 32);
    auto* k0 = ctx->queue_mem.as<unsigned long long>();
    auto* v0 = k0 + n;
    auto* k1 = k0 + 2 * n;
    auto* v1 = k0 + 3 * n;
    {
        LaunchScope ls(ctx, "prepare_ordered", n * 48.0);
        k_prepare_ordered<<<grid_for(n, 256), 256, 0, ctx->stream>>>(cache->view(), dd, drgb, n,
                                                                    ob, k0, v0);
        ls.done();
    }
    sort_pairs_u64(ctx, k0, k1, v0, v1, n, end_bit);
    apply_ordered(ctx, cache, k1, v1, n, ob, d_out, d_slot, d_packed, cache->counters);
}

mcg_status mcg_cache_update_batch(mcg_cache* cache, const mcg_descriptor* d, const float* rgb,
                                  size_t n, int32_t apply_mode, uint8_t* outcome, uint64_t* slot,
                                  uint64_t* packed) {
    return guarded([&] {
        need(cache && d && rgb, "null argument");
        need(cache->world == 1 || cache->stripes, "striped table: attach the stripes first");
        if (!n) return;
        mcg_ctx* ctx = cache->ctx;
        auto* dd = dev_upload(ctx, ctx->scratch_a, d, n);
        auto* dr = dev_upload(ctx, ctx->scratch_b, rgb, 3 * n);
        ctx->scratch_c.ensure(n);
        ctx->scratch_d.ensure(n * 8);
        ctx->scratch_e.ensure(n * 8);
        update_device(cache, dd, dr, n, apply_mode, ctx->scratch_c.as<uint8_t>(),
                      ctx->scratch_d.as<uint64_t>(), ctx->scratch_e.as<uint64_t>());
        dev_download(ctx, outcome, ctx->scratch_c.p, n);
        dev_download(ctx, slot, ctx->scratch_d.p, n);
        dev_download(ctx, packed, ctx->scratch_e.p, n);
        sync(ctx);
    });
}

mcg_status mcg_cache_update_device(mcg_cache* cache, const mcg_descriptor* d_desc,
                                   const float* d_rgb, size_t n, int32_t apply_mode,
                                   uint8_t* d_outcome) {
    return guarded([&] {
        need(cache && d_desc && d_rgb, "null argument");
        update_device(cache, d_desc, d_rgb, n, apply_mode, d_outcome, nullptr, nullptr);
    });
}

mcg_status mcg_cache_lookup_batch(mcg_cache* cache, const mcg_descriptor* d, size_t n,
                                  uint8_t* hit, float* rgb) {
    return guarded([&] {
        need(cache && d && hit && rgb, "null argument");
        need(cache->world == 1 || cache->stripes, "striped table: attach the stripes first");
        if (!n) return;
        mcg_ctx* ctx = cache->ctx;
        auto* dd = dev_upload(ctx, ctx->scratch_a, d, n);
        ctx->scratch_b.ensure(n);
        ctx->scratch_c.ensure(n * 12);
        LaunchScope ls(ctx, "cache_lookup", n * (8.0 * cache->n_entries));
        k_lookup<<<grid_for(n, 256), 256, 0, ctx->stream>>>(cache->view(), dd, n,
                                                           ctx->scratch_b.as<uint8_t>(),
                                                           ctx->scratch_c.as<float>(), cache->counters);
        ls.done();
        dev_download(ctx, hit, ctx->scratch_b.p, n);
        dev_download(ctx, rgb, ctx->scratch_c.p, 3 * n);
        sync(ctx);
    });
}

mcg_status mcg_cache_lookup_device(mcg_cache* cache, const mcg_descriptor* d_desc, size_t n,
                                   uint8_t* d_hit, float* d_rgb) {
    return guarded([&] {
        need(cache && d_desc, "null argument");
        if (!n) return;
        need(cache->world == 1 || cache->stripes, "striped table: attach the stripes first");
        mcg_ctx* ctx = cache->ctx;
        LaunchScope ls(ctx, "cache_lookup", n * (8.0 * cache->n_entries));
        k_lookup<<<grid_for(n, 256), 256, 0, ctx->stream>>>(cache->view(), d_desc, n, d_hit,
                                                           d_rgb, cache->counters);
        ls.done();
    });
}

mcg_status mcg_cache_read_slots(mcg_cache* cache, uint64_t first, size_t n, uint64_t* words) {
    return guarded([&] {
        need(cache && words, "null argument");
        need(first + n <= cache->local_words(), "slot range out of bounds (this stripe's words)");
        if (!n) return;
        read_logical(cache, first, n, words);
    });
}

mcg_status mcg_cache_write_slots(mcg_cache* cache, uint64_t first, size_t n, const uint64_t* words) {
    return guarded([&] {
        need(cache && (words || !n), "null argument");
        need(first + n <= cache->local_words(), "slot range out of bounds (this stripe's words)");
        if (!n) return;
        write_logical(cache, first, n, words);
    });
}

mcg_status mcg_cache_occupied(mcg_cache* cache, uint64_t* occupied) {
    return guarded([&] {
        need(cache && occupied, "null argument");
        mcg_ctx* ctx = cache->ctx;
        cuda_check(cudaMemsetAsync(cache->counters + 7, 0, 8, ctx->stream), "memset");
        const uint64_t n = cache->local_words();   // head and tail arrays
        LaunchScope ls(ctx, "occupied", n * 8.0);
        k_occupied<<<148 * 8, 256, 0, ctx->stream>>>(cache->slots, n, cache->counters + 7);
        ls.done();
        unsigned long long v = 0;
        dev_download(ctx, &v, cache->counters + 7, 1);
        sync(ctx);
        *occupied = v;
    });
}

mcg_status mcg_cache_counters_get(mcg_cache* cache, mcg_cache_counters* out) {
    return guarded([&] {
        need(cache && out, "null argument");
        unsigned long long v[8];
        dev_download(cache->ctx, v, cache->counters, 8);
        sync(cache->ctx);
        out->lookups = v[0];
        out->hits = v[1];
        out->inserts_won = v[2];
        out->inserts_lost_full = v[3];
    });
}

mcg_status mcg_cache_counters_reset(mcg_cache* cache) {
    return guarded([&] {
        need(cache != nullptr, "null cache");
        cuda_check(cudaMemsetAsync(cache->counters, 0, 8 * sizeof(unsigned long long),
                                   cache->ctx->stream), "memset");
        sync(cache->ctx);
    });
}

mcg_status mcg_cache_dump(mcg_cache* cache, const char* path) {
    return guarded([&] {
        need(cache && path, "null argument");
        need(cache->world == 1, "dump of a striped table: dump each stripe's words (mcg_cache_read_slots)");
        std::ofstream out(path, std::ios::binary);
        if (!out) fail(MCG_ERR_IO, std::string("cannot open cache dump for writing: ") + path);
        const uint64_t header[2] = {cache->n_cells, cache->n_entries};
        out.write(reinterpret_cast<const char*>(header), sizeof(header));
        const uint64_t total = cache->n_cells * cache->n_entries;
        const size_t chunk = 1u << 24;
        std::vector<uint64_t> buf(std::min<uint64_t>(total, chunk));
        for (uint64_t off = 0; off < total; off += chunk) {
            const size_t n = static_cast<size_t>(std::min<uint64_t>(chunk, total - off));
            read_logical(cache, off, n, buf.data());
            out.write(reinterpret_cast<const char*>(buf.data()), static_cast<std::streamsize>(n * 8));
        }
        if (!out) fail(MCG_ERR_IO, std::string("short write on cache dump: ") + path);
    });
}

mcg_status mcg_cache_trace_start(mcg_cache* cache, uint64_t capacity) {
    return guarded([&] {
        need(cache != nullptr, "null cache");
        need(capacity > 0 && capacity < (1ull << 34), "trace capacity out of range");
        if (cache->trace) cudaFree(cache->trace);
        cache->trace = nullptr;
        cache->trace_cap = 0;
        cuda_check(cudaMalloc(&cache->trace, capacity * 20), "cudaMalloc(trace)");
        if (!cache->trace_count) cuda_check(cudaMalloc(&cache->trace_count, 8), "cudaMalloc(trace count)");
        cuda_check(cudaMemsetAsync(cache->trace_count, 0, 8, cache->ctx->stream), "memset");
        cache->trace_cap = capacity;
        sync(cache->ctx);
    });
}

mcg_status mcg_cache_trace_stop(mcg_cache* cache, uint64_t* recorded) {
    return guarded([&] {
        need(cache != nullptr, "null cache");
        unsigned long long v = 0;
        if (cache->trace_count) {
            dev_download(cache->ctx, &v, cache->trace_count, 1);
            sync(cache->ctx);
        }
        if (recorded) *recorded = std::min<uint64_t>(v, cache->trace_cap);
        cache->trace_cap = 0;   // recording off; the buffer stays readable
    });
}

mcg_status mcg_cache_trace_read(mcg_cache* cache, uint64_t first, size_t n, mcg_descriptor* out) {
    return guarded([&] {
        need(cache && out, "null argument");
        need(cache->trace != nullptr, "no trace recorded");
        unsigned long long v = 0;
        dev_download(cache->ctx, &v, cache->trace_count, 1);
        sync(cache->ctx);
        need(first + n <= v, "trace range out of bounds");
        if (!n) return;
        dev_download(cache->ctx, reinterpret_cast<uint32_t*>(out), cache->trace + 5 * first, 5 * n);
        sync(cache->ctx);
    });
}

mcg_status mcg_cache_insert_log_start(mcg_cache* cache, uint64_t capacity) {
    return guarded([&] {
        need(cache != nullptr, "null cache");
        need(capacity > 0 && capacity < (1ull << 34), "insert log capacity out of range");
        need(cache->world == 1, "insert log of a striped table");
        if (capacity > cache->ilog_alloc) {
            if (cache->ilog) cudaFree(cache->ilog);
            cache->ilog = nullptr;
            cache->ilog_alloc = 0;
            cuda_check(cudaMalloc(&cache->ilog, capacity * 28), "cudaMalloc(insert log)");
            cache->ilog_alloc = capacity;
        }
        if (!cache->ilog_count) cuda_check(cudaMalloc(&cache->ilog_count, 8), "cudaMalloc(insert log count)");
        cuda_check(cudaMemsetAsync(cache->ilog_count, 0, 8, cache->ctx->stream), "memset");
        cache->ilog_cap = capacity;
        sync(cache->ctx);
    });
}

mcg_status mcg_cache_insert_log_stop(mcg_cache* cache, uint64_t* won) {
    return guarded([&] {
        need(cache != nullptr, "null cache");
        unsigned long long v = 0;
        if (cache->ilog_count) {
            dev_download(cache->ctx, &v, cache->ilog_count, 1);
            sync(cache->ctx);
        }
        if (won) *won = v;   // may exceed the capacity: then only `capacity` records were kept
        cache->ilog_cap = 0;
    });
}

mcg_status mcg_cache_insert_log_read(mcg_cache* cache, uint64_t first, size_t n, mcg_insert_record* out) {
    return guarded([&] {
        need(cache && (out || !n), "null argument");
        need(cache->ilog != nullptr, "no insert log recorded");
        unsigned long long v = 0;
        dev_download(cache->ctx, &v, cache->ilog_count, 1);
        sync(cache->ctx);
        need(first + n <= std::min<uint64_t>(v, cache->ilog_alloc), "insert log range out of bounds");
        if (!n) return;
        static_assert(sizeof(mcg_insert_record) == 28, "mcg_insert_record layout");
        std::vector<uint32_t> raw(7 * n);
        dev_download(cache->ctx, raw.data(), cache->ilog + 7 * first, 7 * n);
        sync(cache->ctx);
        for (size_t i = 0; i < n; ++i) {
            const uint32_t* r = raw.data() + 7 * i;
            mcg_insert_record& o = out[i];
            std::memset(&o, 0, sizeof(o));
            o.desc.mat_idx = r[0];
            o.desc.node_idx = r[1];
            o.desc.mip_level = static_cast<uint8_t>(r[2]);
            o.desc.texel_x = r[3];
            o.desc.texel_y = r[4];
            o.entry = r[5];
            o.payload = r[6];
        }
    });
}

mcg_status mcg_probe_replay(mcg_cache* cache, const mcg_descriptor* d, uint64_t n, int32_t blocks_per_sm,
                            double* ms_out, double* bytes_out, mcg_cache_counters* counters) {
    return guarded([&] {
        need(cache && d, "null argument");
        need(cache->world == 1 || cache->stripes, "striped table: attach the stripes first");
        if (!n) return;
        mcg_ctx* ctx = cache->ctx;
        auto* dd = dev_upload(ctx, ctx->scratch_a, d, n);
        cudaEvent_t a = take_event(ctx), b = take_event(ctx);
        cuda_check(cudaMemsetAsync(cache->counters, 0, 8 * sizeof(unsigned long long), ctx->stream), "memset");
        cudaEventRecord(a, ctx->stream);
        {
            LaunchScope ls(ctx, "probe_replay", 0.0);
            // blocks_per_sm < 0: the software-pipelined kernel (measured slower on
            // a render's trace, whose coherent lookups mostly hit L2: 34.4 vs
            // 37.3 G probes/s, profiles/README.md)
            const bool pipe = blocks_per_sm < 0;
            const int bps = blocks_per_sm < 0 ? -blocks_per_sm : blocks_per_sm;
            const unsigned grid = 148u * static_cast<unsigned>(bps > 0 ? bps : 8);
            if (pipe) k_probe_replay<true><<<grid, 256, 0, ctx->stream>>>(cache->view(), dd, n, cache->counters);
            else k_probe_replay<false><<<grid, 256, 0, ctx->stream>>>(cache->view(), dd, n, cache->counters);
            ls.done();
        }
        cudaEventRecord(b, ctx->stream);
        cuda_check(cudaEventSynchronize(b), "probe replay");
        float ms = 0.0f;
        cudaEventElapsedTime(&ms, a, b);
        ctx->event_pool.push_back(a);
        ctx->event_pool.push_back(b);
        unsigned long long v[8];
        dev_download(ctx, v, cache->counters, 8);
        sync(ctx);
        if (ms_out) *ms_out = ms;
        // 8*Ne per lookup, 8*Ne per insert attempt (the miss's scan is the lookup's), +8 per won CAS
        if (bytes_out) *bytes_out = static_cast<double>(v[0]) * 8.0 * cache->n_entries + static_cast<double>(v[2]) * 8.0;
        if (counters) {
            counters->lookups = v[0];
            counters->hits = v[1];
            counters->inserts_won = v[2];
            counters->inserts_lost_full = v[3];
        }
    });
}

mcg_status mcg_probe_bench(mcg_cache* cache, uint64_t n, uint64_t seed, int32_t phase,
                           int32_t iters, double* ms_out, double* bytes_out) {
    return guarded([&] {
        need(cache != nullptr, "null cache");
        need((phase & 15) <= 2 && ((phase >> 4) & 15) <= 11,
             "phase must be 0, 1 or 2 (+16 * variant, +256 * blocks per SM)");
        mcg_ctx* ctx = cache->ctx;
        cudaEvent_t a = take_event(ctx), b = take_event(ctx);
        cuda_check(cudaMemsetAsync(cache->counters, 0, 8 * sizeof(unsigned long long), ctx->stream), "memset");
        cudaEventRecord(a, ctx->stream);
        const int reps = std::max(1, iters);
        for (int r = 0; r < reps; ++r) {
            LaunchScope ls(ctx, "probe_bench", 0.0);
            const int variant = (phase >> 4) & 15, ph = phase & 15;
            const int per_sm = (phase >> 8) ? (phase >> 8) : 8;   // blocks per SM
            const unsigned grid = 148u * static_cast<unsigned>(per_sm);
            const bool coop = cache->n_entries % 2 == 0 && cache->n_entries <= 10;
            if (variant == 5 && coop) {
                k_probe_bench_pipe<2><<<grid, 256, 0, ctx->stream>>>(cache->view(), n, seed, ph, cache->counters);
            } else if (variant == 6 && coop) {
                k_probe_bench_pipe<4><<<grid, 256, 0, ctx->stream>>>(cache->view(), n, seed, ph, cache->counters);
            } else if (variant == 8 && coop) {
                k_probe_bench_pipe<1, true><<<grid, 256, 0, ctx->stream>>>(cache->view(), n, seed, ph, cache->counters);
            } else if (variant == 9 && coop) {
                k_probe_bench_pipe<2, true><<<grid, 256, 0, ctx->stream>>>(cache->view(), n, seed, ph, cache->counters);
            } else if (variant == 10 && coop) {
                k_probe_bench_pipe<1, false, true><<<grid, 256, 0, ctx->stream>>>(cache->view(), n, seed, ph, cache->counters);
            } else if (variant == 11 && coop) {
                k_probe_bench_pipe<2, false, true><<<grid, 256, 0, ctx->stream>>>(cache->view(), n, seed, ph, cache->counters);
            } else if (variant == 7 && coop) {
                k_probe_bench_pipe<1><<<grid, 256, 0, ctx->stream>>>(cache->view(), n, seed, ph, cache->counters);
            } else if (variant == 4 && coop) {
                k_probe_bench<4><<<grid, 256, 0, ctx->stream>>>(cache->view(), n, seed, ph, cache->counters);
            } else if (variant == 2 && cache->n_entries == 10) {
                k_probe_bench<2><<<grid, 256, 0, ctx->stream>>>(cache->view(), n, seed, ph, cache->counters);
            } else if (variant == 1) {
                k_probe_bench<1><<<grid, 256, 0, ctx->stream>>>(cache->view(), n, seed, ph, cache->counters);
            } else if (variant == 3) {
                k_probe_bench<3><<<grid, 256, 0, ctx->stream>>>(cache->view(), n, seed, ph, cache->counters);
            } else {
                k_probe_bench<0><<<grid, 256, 0, ctx->stream>>>(cache->view(), n, seed, ph, cache->counters);
            }
            ls.done();
        }
        cudaEventRecord(b, ctx->stream);
        cuda_check(cudaEventSynchronize(b), "probe bench");
        float ms = 0.0f;
        cudaEventElapsedTime(&ms, a, b);
        ctx->event_pool.push_back(a);
        ctx->event_pool.push_back(b);
        unsigned long long v[8];
        dev_download(ctx, v, cache->counters, 8);
        sync(ctx);
        // 8*Ne bytes per lookup and per insert attempt, +8 per won CAS.
        const double cellb = 8.0 * cache->n_entries;
        if (ms_out) *ms_out = ms / reps;
        if (bytes_out) *bytes_out = (static_cast<double>(v[0]) * cellb + static_cast<double>(v[5]) * cellb +
                                     static_cast<double>(v[2]) * 8.0) / reps;
    });
}

// ---- scene upload & per-point execution -----------------------------------

mcg_status mcg_upload_scene(mcg_ctx* ctx, const mcg_scene* scene) {
    if (ctx && !ctx->peers.empty()) {
        // every device of a multi-device context holds the scene
        for (mcg_ctx* p : ctx->peers) {
            const mcg_status st = mcg_upload_scene(p, scene);
            if (st != MCG_OK) return st;
        }
    }
    return guarded([&] {
        need(ctx && scene, "null argument");
        cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
        mcg_flat_scene f;
        const mcg_status s = mcg_scene_flat(scene, &f);
        if (s != MCG_OK) fail(s, mcg_last_error());
        DeviceScene& D = ctx->scene;
        D.reset();
        if (D.bufs.size() < 20) D.bufs.resize(20);
        auto up = [&](int k, const void* p, size_t bytes) -> const void* {
            D.bufs[k].ensure(std::max<size_t>(bytes, 16));
            if (bytes) cuda_check(cudaMemcpyAsync(D.bufs[k].p, p, bytes, cudaMemcpyHostToDevice, ctx->stream), "H2D scene");
            return D.bufs[k].p;
        };
        mcgd::SceneView& v = D.view;
        v.prim_geom = static_cast<const float4*>(up(0, f.prim_geom, f.n_prims * 48ull));
        v.prim_uv = static_cast<const float2*>(up(1, f.prim_uv, f.n_prims * 24ull));
        v.prim_info = static_cast<const uint32_t*>(up(2, f.prim_info, f.n_prims * 4ull));
        v.nodes = static_cast<const float4*>(up(3, f.nodes, f.n_nodes * sizeof(mcg_bvh_node)));
        v.n_nodes = f.n_nodes;
        // Child-pair layout: internal node i holds both children's boxes and
        // references (an internal child by its node index, a leaf by
        // (~first, count)), so one 64-byte fetch tests both child boxes (the
        // traversal still visits nodes in the reference's order, see
        // mcg_render.cu traverse_closest).
        std::vector<mcg_bvh_node> pairs(2 * static_cast<size_t>(std::max<uint32_t>(f.n_nodes, 1)));
        for (uint32_t i = 0; i < f.n_nodes; ++i) {
            const mcg_bvh_node& nd = f.nodes[i];
            if (nd.a < 0) continue;
            const int32_t child[2] = {nd.a, nd.b};
            for (int k = 0; k < 2; ++k) {
                mcg_bvh_node c = f.nodes[child[k]];
                if (c.a >= 0) {
                    c.a = child[k];
                    c.b = 0;
                }
                pairs[2 * i + k] = c;
            }
        }
        v.pairs = static_cast<const float4*>(up(14, pairs.data(), f.n_nodes * 2 * sizeof(mcg_bvh_node)));
        // W-wide nodes (W = mcgd::kClosestWidth, 4 or 8): each holds the
        // descendants log2(W) levels below a reference node (a leaf above
        // that depth stands for itself), in left-to-right order, so a LIFO
        // stack still visits in the reference's order; the skipped boxes
        // contain their children's boxes, so their culling is implied
        // (DESIGN.md §5).
        const int W = mcgd::kClosestWidth;
        int depth_levels = 0;
        while ((1 << depth_levels) < W) ++depth_levels;
        std::vector<mcg_bvh_node> quads;
        std::function<int32_t(int32_t)> collapse = [&](int32_t x) -> int32_t {
            const int32_t q = static_cast<int32_t>(quads.size() / W);
            quads.resize(quads.size() + W, mcg_bvh_node{{0, 0, 0}, 0, {0, 0, 0}, 0});
            std::vector<int32_t> entries{f.nodes[x].a, f.nodes[x].b};
            for (int level = 1; level < depth_levels; ++level) {
                std::vector<int32_t> next;
                for (int32_t e : entries) {
                    if (f.nodes[e].a < 0) {
                        next.push_back(e);
                    } else {
                        next.push_back(f.nodes[e].a);
                        next.push_back(f.nodes[e].b);
                    }
                }
                entries.swap(next);
            }
            int k = 0;
            for (int32_t e : entries) {
                mcg_bvh_node rec = f.nodes[e];
                if (rec.a >= 0) {
                    rec.a = collapse(e);
                    rec.b = -1;
                }
                quads[static_cast<size_t>(W) * q + k++] = rec;
            }
            return q;
        };
        v.root_a = 0;
        v.root_b = 0;
        if (f.n_nodes) {
            std::memcpy(D.root_lo, f.nodes[0].lo, sizeof(D.root_lo));
            std::memcpy(D.root_hi, f.nodes[0].hi, sizeof(D.root_hi));
            if (f.nodes[0].a < 0) {
                v.root_a = f.nodes[0].a;
                v.root_b = f.nodes[0].b;
            } else {
                collapse(0);
                v.root_a = 0;
                v.root_b = -1;
            }
        }
        v.quads = static_cast<const float4*>(up(15, quads.data(), quads.size() * sizeof(mcg_bvh_node)));
        // Worst-case stack of the LIFO traversal: a node pushes its k
        // entries and descends into one of them, leaving k-1 behind.
        auto stack_need = [](const std::vector<mcg_bvh_node>& qs, int width) -> uint32_t {
            const size_t nq = qs.size() / width;
            std::vector<uint32_t> need(nq, 1);
            for (size_t q = nq; q-- > 0;) {
                uint32_t k = 0, deepest = 1;
                for (int e = 0; e < width; ++e) {
                    const mcg_bvh_node& r = qs[width * q + e];
                    if (r.b == 0) continue;
                    ++k;
                    if (r.b < 0) deepest = std::max(deepest, need[r.a]);
                }
                need[q] = std::max(k, (k ? k - 1 : 0) + deepest);
            }
            return nq ? std::max<uint32_t>(1, need[0]) : 1;
        };
        D.max_stack4 = stack_need(quads, W);
        if (D.max_stack4 > 63) fail(MCG_ERR_INVALID_ARGUMENT, "BVH too deep for the traversal stack");
        // Shadow tree: the reference's leaves (their exact boxes and
        // primitive ranges) regrouped by a binned SAH build. Any-hit is a
        // boolean: a triangle is found iff its leaf's box passes and the
        // triangle test hits (every ancestor box contains the leaf box, and
        // the slab test is monotone, so ancestors never reject first) -- so
        // any hierarchy over the same leaves answers exactly as the
        // reference's tree does.
        // MCG_SHADOW_BUILD=host: the host builder; default: the same SAH
        // tree built on the device (mcg_build.cu)
        std::vector<mcg_bvh_node> squads;
        const char* sb_env = std::getenv("MCG_SHADOW_BUILD");
        if (sb_env && std::string(sb_env) == "host") {
            squads = build_shadow_tree(f, mcgd::kShadowWidth, v.sroot_a, v.sroot_b);
        } else {
            std::vector<mcg_bvh_node> leaves;
            const mcg_bvh_node* rn = static_cast<const mcg_bvh_node*>(f.nodes);
            for (uint32_t i = 0; i < f.n_nodes; ++i)
                if (rn[i].a < 0) leaves.push_back(rn[i]);
            squads = build_shadow_tree_device(ctx, leaves, mcgd::kShadowWidth, v.sroot_a, v.sroot_b);
        }
        D.max_stack_s = stack_need(squads, mcgd::kShadowWidth);
        D.shadow_nodes = squads;
        if (D.max_stack_s > 63) fail(MCG_ERR_INVALID_ARGUMENT, "shadow BVH too deep for the traversal stack");
        v.squads = static_cast<const float4*>(up(16, squads.data(), squads.size() * sizeof(mcg_bvh_node)));
        // The same 4-wide nodes transposed (mcg_device.cuh, closest_q4): eight
        // float4 rows -- lo.x, lo.y, lo.z, hi.x, hi.y, hi.z of the four entries,
        // then their a and b words -- so the traversal tests four boxes with
        // packed f32x2 arithmetic and picks near/far planes by address.
        auto transpose4 = [](const std::vector<mcg_bvh_node>& aos) {
            std::vector<float> soa(aos.size() / 4 * 32, 0.0f);
            for (size_t q = 0; q < aos.size() / 4; ++q) {
                float* row = soa.data() + 32 * q;
                for (int e = 0; e < 4; ++e) {
                    const mcg_bvh_node& r = aos[4 * q + e];
                    row[0 + e] = r.lo[0];
                    row[4 + e] = r.lo[1];
                    row[8 + e] = r.lo[2];
                    row[12 + e] = r.hi[0];
                    row[16 + e] = r.hi[1];
                    row[20 + e] = r.hi[2];
                    std::memcpy(row + 24 + e, &r.a, 4);
                    std::memcpy(row + 28 + e, &r.b, 4);
                }
            }
            return soa;
        };
        if (mcgd::kClosestWidth == 4) {
            const std::vector<float> qs = transpose4(quads);
            v.quads_soa = static_cast<const float4*>(up(17, qs.data(), qs.size() * sizeof(float)));
        }
        if (mcgd::kShadowWidth == 4) {
            const std::vector<float> ss = transpose4(squads);
            v.squads_soa = static_cast<const float4*>(up(18, ss.data(), ss.size() * sizeof(float)));
        }
        v.plights = static_cast<const mcg_point_light*>(up(4, f.point_lights, f.n_point_lights * sizeof(mcg_point_light)));
        v.n_plights = f.n_point_lights;
        v.rlights = static_cast<const mcg_rect_light*>(up(5, f.rect_lights, f.n_rect_lights * sizeof(mcg_rect_light)));
        v.n_rlights = f.n_rect_lights;
        v.programs = static_cast<const mcg_program*>(up(6, f.programs, f.n_programs * sizeof(mcg_program)));
        v.n_programs = f.n_programs;
        // one spare word past the last program: the VM fetches pc + 1 ahead
        D.bufs[7].ensure((f.n_code + 1) * sizeof(mcg_insn));
        v.code = static_cast<const mcg_insn*>(up(7, f.code, f.n_code * sizeof(mcg_insn)));
        v.n_code = f.n_code;
        // The look-ahead table: per program, its cache points with bracket
        // < kAhead (CacheLookup node, uses_uv flag, bracket index in bits
        // 16-23), largest subtree (skip_offset) first: the first two give
        // the sort key's hit bits, so warps are uniform on the brackets that
        // cost the most (MCG_AHEAD_ORDER=bracket: bracket order).
        {
            const char* ao_env = std::getenv("MCG_AHEAD_ORDER");
            const bool by_size = !(ao_env && std::string(ao_env) == "bracket");
            std::vector<uint2> acp(static_cast<size_t>(f.n_programs) * mcgd::kAhead, make_uint2(0u, 0u));
            for (uint32_t i = 0; i < f.n_programs; ++i) {
                const mcg_program& pr = f.programs[i];
                std::vector<std::pair<int32_t, uint2>> cps;   // (-subtree size, entry)
                for (uint32_t c = 0; c < pr.code_len; ++c) {
                    const mcg_insn& in = f.code[pr.code_offset + c];
                    if (in.op == MCG_OP_CACHE_LOOKUP && in.bracket < mcgd::kAhead) {
                        const uint2 e = make_uint2(in.arg, (in.flags & MCG_F_USES_UV) | mcgd::kAheadValid |
                                                               (static_cast<uint32_t>(in.bracket) << 16));
                        cps.push_back({by_size ? -in.imm.i : static_cast<int32_t>(in.bracket), e});
                    }
                }
                std::stable_sort(cps.begin(), cps.end(),
                                 [](const auto& a, const auto& b) { return a.first < b.first; });
                for (size_t k = 0; k < cps.size() && k < mcgd::kAhead; ++k) acp[i * mcgd::kAhead + k] = cps[k].second;
            }
            v.ahead_cp = static_cast<const uint2*>(up(19, acp.data(), acp.size() * sizeof(uint2)));
        }
        v.consts = static_cast<const mcg_const*>(up(8, f.consts, f.n_consts * sizeof(mcg_const)));
        v.noise = static_cast<const mcg_noise*>(up(9, f.noise, f.n_noise * sizeof(mcg_noise)));
        v.ramps = static_cast<const mcg_ramp*>(up(10, f.ramps, f.n_ramps * sizeof(mcg_ramp)));
        v.stops = static_cast<const mcg_ramp_stop*>(up(11, f.ramp_stops, f.n_ramp_stops * sizeof(mcg_ramp_stop)));
        v.textures = static_cast<const mcg_texture*>(up(12, f.textures, f.n_textures * sizeof(mcg_texture)));
        v.texels = static_cast<const float4*>(up(13, f.texels, f.n_texels * 16ull));
        std::memcpy(v.env, f.env, sizeof(v.env));
        D.max_stack = 1;
        D.max_cache_points = 0;
        for (uint32_t i = 0; i < f.n_programs; ++i) {
            D.max_stack = std::max(D.max_stack, f.programs[i].max_stack);
            D.max_cache_points = std::max(D.max_cache_points, f.programs[i].cache_point_count);
        }
        D.cam = f;
        D.cam.prim_geom = nullptr;  // only camera/env fields are used later
        D.loaded = true;
        sync(ctx);
    });
}

mcg_status mcg_shadow_tree(mcg_ctx* ctx, mcg_bvh_node* out, size_t cap, size_t* n_out, int32_t* root_a,
                           int32_t* root_b) {
    return guarded([&] {
        need(ctx && n_out && root_a && root_b, "null argument");
        need(ctx->scene.loaded, "no scene uploaded");
        const std::vector<mcg_bvh_node>& t = ctx->scene.shadow_nodes;
        *n_out = t.size() / mcgd::kShadowWidth;
        *root_a = ctx->scene.view.sroot_a;
        *root_b = ctx->scene.view.sroot_b;
        if (out && cap >= t.size()) std::memcpy(out, t.data(), t.size() * sizeof(mcg_bvh_node));
    });
}

mcg_status mcg_execute_batch(mcg_ctx* ctx, uint32_t slot, const float* sp, size_t n,
                             mcg_cache* cache, int32_t cache_mode, int32_t mip_offset,
                             float* values, uint32_t* nodes_found, uint32_t* instructions) {
    return guarded([&] {
        need(ctx && sp && values && nodes_found && instructions, "null argument");
        need(ctx->scene.loaded, "no scene uploaded");
        need(slot < ctx->scene.view.n_programs, "material slot out of range");
        if (!n) return;
        const bool cache_on = cache != nullptr && cache_mode != MCG_CACHE_OFF;
        const bool deferred = cache_on && cache_mode == MCG_CACHE_DETERMINISTIC;
        auto* dsp = dev_upload(ctx, ctx->scratch_a, sp, 15 * n);
        ctx->scratch_b.ensure(n * 16);
        ctx->scratch_c.ensure(n * 4);
        ctx->scratch_d.ensure(n * 4);
        const int block = 128;
        const int max_stack = static_cast<int>(ctx->scene.max_stack);
        const size_t smem = static_cast<size_t>(max_stack) * block * 3 * sizeof(float);
        if (cache && cache->world > 1 && !cache->stripes) fail(MCG_ERR_INVALID_ARGUMENT, "striped table: attach the stripes first");
        mcgd::CacheView cv = cache ? cache->view() : mcgd::CacheView{nullptr, nullptr, 1, ~0ull, 1, 1, 1, nullptr, nullptr, nullptr, 0};
        unsigned long long* counters = cache ? cache->counters : ctx->stats_mem.as<unsigned long long>();
        mcgd::StoreQueue q{nullptr, nullptr, nullptr, 0};
        const uint64_t cap = deferred ? n * std::max<uint32_t>(1, ctx->scene.max_cache_points) : 0;
        if (deferred) {
            ctx->queue_mem.ensure(cap * 32 + 64);
            q.keys = ctx->queue_mem.as<unsigned long long>();
            q.vals = q.keys + cap;
            q.count = reinterpret_cast<unsigned int*>(q.keys + 4 * cap);
            q.capacity = static_cast<unsigned>(cap);
            cuda_check(cudaMemsetAsync(q.count, 0, 4, ctx->stream), "memset");
        }
        {
            LaunchScope ls(ctx, "execute", 0.0);
            if (deferred) {
                cudaFuncSetAttribute(k_execute<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
                k_execute<true><<<grid_for(n, block), block, smem, ctx->stream>>>(
                    ctx->scene.view, cv, 1, mip_offset, slot, dsp, n, max_stack,
                    ctx->scratch_b.as<float>(), ctx->scratch_c.as<uint32_t>(),
                    ctx->scratch_d.as<uint32_t>(), q, counters);
            } else {
                cudaFuncSetAttribute(k_execute<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
                k_execute<false><<<grid_for(n, block), block, smem, ctx->stream>>>(
                    ctx->scene.view, cv, cache_on ? 1 : 0, mip_offset, slot, dsp, n, max_stack,
                    ctx->scratch_b.as<float>(), ctx->scratch_c.as<uint32_t>(),
                    ctx->scratch_d.as<uint32_t>(), q, counters);
            }
            ls.done();
        }
        if (deferred) {
            unsigned int count = 0;
            dev_download(ctx, &count, q.count, 1);
            sync(ctx);
            need(count <= cap, "store queue overflow");
            const int ob = std::max(1, bits_for((static_cast<uint64_t>(n) << 6) - 1));
            // Re-key (cell << 32 | order) -> (cell << ob | order) is implicit:
            // order keys already fit in the low 32 bits, cells in the high 32.
            auto* k1 = q.keys + 2 * cap;
            auto* v1 = q.keys + 3 * cap;
            sort_pairs_u64(ctx, q.keys, k1, q.vals, v1, count, 64);
            apply_ordered(ctx, cache, k1, v1, count, 32, nullptr, nullptr, nullptr, cache->counters);
            (void)ob;
        }
        dev_download(ctx, values, ctx->scratch_b.p, 4 * n);
        dev_download(ctx, nodes_found, ctx->scratch_c.p, n);
        dev_download(ctx, instructions, ctx->scratch_d.p, n);
        sync(ctx);
    });
}

}  // extern "C"

// Device-side building blocks shared by the runtime and render translation
// units: the HBM table probe/insert (cache.cpp:94-136) and the warp-uniform
// stack-machine interpreter (stackvm.cpp:248-368).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "device_math.cuh"

namespace mcgd {

constexpr unsigned kFull = 0xffffffffu;

// ---------------------------------------------------------------------------
// Table view
// ---------------------------------------------------------------------------
struct CacheView {
    uint64_t* slots;          // head words: n_cells x head_n, cell-major
    uint64_t* tail;           // tail words: n_cells x (n_entries - head_n), or null
    uint64_t n_cells;
    uint64_t magic;           // floor((2^64-1) / n_cells) for fast_mod
    uint32_t n_entries;
    uint32_t head_n;          // a cell's first min(n_entries, 8) slots: one 64-byte DRAM block
    uint32_t world;           // > 1: one logical table striped by cell over `world` devices
    uint64_t* const* stripes; // (head, tail) device pointers of every stripe (peer memory over NVLink)
    uint32_t* trace;          // optional descriptor log: 5 words per lookup (mcg_descriptor)
    unsigned long long* trace_count;
    uint64_t trace_cap;
    uint32_t* ilog;           // optional log of won inserts: 7 words each (mcg_insert_record)
    unsigned long long* ilog_count;
    uint64_t ilog_cap;
};

// Appends a won insert (descriptor, entry within the cell, payload) to the
// table's insert log, when one is recording (mcg_cache_insert_log_*): the
// host drop-in replays these through the caller's MaterialCache::update so
// the host table, its counters and its dump follow the device's.
__device__ __forceinline__ void log_insert(const CacheView& c, uint32_t mat, uint32_t node, uint32_t mip,
                                           uint32_t tx, uint32_t ty, uint32_t entry, uint32_t payload) {
    const unsigned long long at = atomicAdd(c.ilog_count, 1ull);
    if (at >= c.ilog_cap) return;
    uint32_t* r = c.ilog + 7 * at;
    r[0] = mat;
    r[1] = node;
    r[2] = mip;
    r[3] = tx;
    r[4] = ty;
    r[5] = entry;
    r[6] = payload;
}

// Where a cell's slots live. DRAM serves random reads in 64-byte blocks, and
// an 80-byte cell always straddles two of them (ncu: 142 B of DRAM per
// lookup); so a cell of more than 8 slots keeps its first 8 in a 64-byte
// aligned head array and the rest in a tail array. The scan reads the head
// (one block) and touches the tail only when the head neither matched nor
// held an empty slot. Slot indices stay the logical cell * n_entries + e.
// A striped table keeps cell c on stripe c % world at local cell c / world,
// so every device sees the same logical table.
__device__ __forceinline__ uint64_t* head_words(const CacheView& c, uint64_t cell) {
    MCG_CHECK(cell < c.n_cells);
    if (c.world <= 1u) return c.slots + cell * c.head_n;
    return c.stripes[2 * (cell % c.world)] + (cell / c.world) * c.head_n;
}
__device__ __forceinline__ uint64_t* tail_words(const CacheView& c, uint64_t cell) {
    const uint32_t tn = c.n_entries - c.head_n;
    if (c.world <= 1u) return c.tail + cell * tn;
    return c.stripes[2 * (cell % c.world) + 1] + (cell / c.world) * tn;
}
__device__ __forceinline__ uint64_t* slot_ptr(const CacheView& c, uint64_t cell, uint32_t e) {
    MCG_CHECK(cell < c.n_cells && e < c.n_entries);
    return e < c.head_n ? head_words(c, cell) + e : tail_words(c, cell) + (e - c.head_n);
}
// Result of scanning one cell as lookup() does (cache.cpp:121-136): a match,
// or the first empty slot (where update() would CAS, cache.cpp:108), or a
// full cell (update() -> CellFull).
struct Probe {
    uint32_t payload;
    int32_t where;   // hit: matching slot; miss: first empty slot; -1: cell full
    bool hit;
};

// One step of the reference scan (cache.cpp:127-134 / :99-116): an empty slot
// ends it (miss, update() would CAS there), a matching check-hash is a hit.
__device__ __forceinline__ bool scan_word(uint64_t w, int32_t idx, uint32_t check, Probe& r) {
    if (w == 0ull) {
        r.where = idx;
        return true;
    }
    if (static_cast<uint32_t>(w >> 32) == check) {
        r.hit = true;
        r.where = idx;
        r.payload = static_cast<uint32_t>(w);
        return true;
    }
    return false;
}

// Scans a cell with 128-bit loads. kFirstPairs 16-byte pairs are fetched
// before the first decision and the rest (cells up to Ne = 10 live in
// registers) in one more round trip: kFirstPairs = 1 reads one DRAM sector
// when the scan ends early (sparse tables), kFirstPairs = 5 fetches the whole
// 80-byte cell at once (one round trip, full tables). Loads bypass L1
// (ld.global.cg) so concurrent inserts from other SMs are seen as soon as L2
// sees them.
template <int kFirstPairs>
__device__ __forceinline__ Probe probe_cell_t(const CacheView& c, uint64_t cell_index, uint32_t check) {
    Probe r{0u, -1, false};
    const uint32_t ne = c.n_entries, hn = c.head_n, tn = ne - hn;
    const uint64_t* cell = head_words(c, cell_index);
    uint32_t i = 0;
    if ((reinterpret_cast<uintptr_t>(cell) & 15u) == 0u && hn >= 2 && hn <= 8 && (hn & 1u) == 0u) {
        const uint32_t npairs = hn >> 1;
        const ulonglong2* p = reinterpret_cast<const ulonglong2*>(cell);
        // the tail's first pair joins the head's second round trip
        // (16-byte aligned when the tail holds an even number of slots)
        const ulonglong2* tp = (tn >= 2 && (tn & 1u) == 0u)
                                   ? reinterpret_cast<const ulonglong2*>(tail_words(c, cell_index))
                                   : nullptr;
        ulonglong2 w[5];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (k < kFirstPairs && k < static_cast<int>(npairs)) w[k] = __ldcg(p + k);
        }
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            if (k >= static_cast<int>(npairs) + (tp ? 1 : 0)) break;
            if (k == kFirstPairs) {
#pragma unroll
                for (int j = kFirstPairs; j < 5; ++j) {
                    if (j < static_cast<int>(npairs)) w[j] = __ldcg(p + j);
                    else if (j == static_cast<int>(npairs) && tp) w[j] = __ldcg(tp);
                }
            }
            if (k == static_cast<int>(npairs) && k < kFirstPairs) w[k] = __ldcg(tp);
            if (scan_word(w[k].x, 2 * k, check, r) || scan_word(w[k].y, 2 * k + 1, check, r)) return r;
        }
        i = tp ? hn + 2 : hn;
    }
    for (; i < hn; ++i) {
        if (scan_word(__ldcg(cell + i), static_cast<int32_t>(i), check, r)) return r;
    }
    if (ne > hn) {
        const uint64_t* t = tail_words(c, cell_index);
        for (uint32_t j = (i > hn ? i - hn : 0u); j < tn; ++j) {
            if (scan_word(__ldcg(t + j), static_cast<int32_t>(hn + j), check, r)) return r;
        }
    }
    return r;  // full, no match
}

#ifndef MCG_VM_FIRST_PAIRS
#define MCG_VM_FIRST_PAIRS 1   // 16-byte pairs the VM's probe reads before its first decision
#endif
__device__ __forceinline__ Probe probe_cell(const CacheView& c, uint64_t cell, uint32_t check) {
    return probe_cell_t<1>(c, cell, check);
}

// Two-round scan aligned to 64-byte DRAM blocks: round one reads from the
// cell start to the end of its first 64-byte block (2..8 words, one block),
// round two the rest of the cell (at most one more block for Ne <= 10). A
// scan that ends in round one costs one block; a full scan two -- never the
// three blocks an 80-byte cell can straddle.
__device__ __forceinline__ Probe probe_cell_blk(const CacheView& c, uint64_t cell_index, uint32_t check) {
    Probe r{0u, -1, false};
    const uint32_t ne = c.n_entries;
    const uint64_t* cell = head_words(c, cell_index);
    if ((reinterpret_cast<uintptr_t>(cell) & 15u) != 0u || ne > 10 || c.head_n != ne) {
        return probe_cell_t<1>(c, cell_index, check);
    }
    const uint32_t npairs = ne >> 1;
    const ulonglong2* p = reinterpret_cast<const ulonglong2*>(cell);
    // pairs in the first 64-byte block: (64 - (addr % 64)) / 16
    const uint32_t first = (64u - static_cast<uint32_t>(reinterpret_cast<uintptr_t>(cell) & 63u)) >> 4;
    ulonglong2 w[5];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if (k < static_cast<int>(first) && k < static_cast<int>(npairs)) w[k] = __ldcg(p + k);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if (k >= static_cast<int>(first) || k >= static_cast<int>(npairs)) break;
        if (scan_word(w[k].x, 2 * k, check, r) || scan_word(w[k].y, 2 * k + 1, check, r)) return r;
    }
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        if (k >= static_cast<int>(first) && k < static_cast<int>(npairs)) w[k] = __ldcg(p + k);
    }
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        if (k < static_cast<int>(first)) continue;
        if (k >= static_cast<int>(npairs)) break;
        if (scan_word(w[k].x, 2 * k, check, r) || scan_word(w[k].y, 2 * k + 1, check, r)) return r;
    }
    for (uint32_t i = 2 * npairs; i < ne; ++i) {
        if (scan_word(__ldcg(cell + i), static_cast<int32_t>(i), check, r)) return r;
    }
    return r;
}

// Warp-cooperative probe of up to 32 cells (one per lane of `mask`, n_entries
// <= 32): each round the warp reads floor(32/Ne) whole cells with one 8-byte
// load per lane (each cell one coalesced 8*Ne-byte access), all rounds issued
// before any decision; per cell, ballots over its lanes give the first empty
// slot and the first matching check-hash, i.e. the reference scan.
template <int kNe>
__device__ __forceinline__ Probe probe_warp(const CacheView& c, uint64_t cell, uint32_t check,
                                            bool valid) {
    constexpr int kPer = 32 / kNe;
    constexpr int kRounds = (32 + kPer - 1) / kPer;
    const int lane = static_cast<int>(threadIdx.x & 31u);
    const int g = lane / kNe, word = lane - g * kNe;
    uint64_t w[kRounds];
#pragma unroll
    for (int rd = 0; rd < kRounds; ++rd) {
        const int owner = rd * kPer + g;
        const uint64_t oc = __shfl_sync(kFull, cell, owner & 31);
        const bool ov = __shfl_sync(kFull, valid, owner & 31);
        w[rd] = (g < kPer && owner < 32 && ov) ? __ldcg(slot_ptr(c, oc, static_cast<uint32_t>(word))) : ~0ull;
    }
    Probe mine{0u, -1, false};
#pragma unroll
    for (int rd = 0; rd < kRounds; ++rd) {
#pragma unroll
        for (int gg = 0; gg < kPer; ++gg) {
            const int owner = rd * kPer + gg;
            if (owner >= 32) break;
            const uint32_t chk = __shfl_sync(kFull, check, owner);
            const unsigned gm = ((1u << kNe) - 1u) << (gg * kNe);
            const unsigned empty = __ballot_sync(kFull, w[rd] == 0ull) & gm;
            const unsigned match = __ballot_sync(kFull, static_cast<uint32_t>(w[rd] >> 32) == chk) & gm;
            const uint32_t pay = __shfl_sync(kFull, static_cast<uint32_t>(w[rd]),
                                             match ? __ffs(match) - 1 : 0);
            if (lane == owner) {
                const int fe = empty ? __ffs(empty) - 1 - gg * kNe : kNe;
                const int fm = match ? __ffs(match) - 1 - gg * kNe : kNe;
                if (fm < fe) {
                    mine.hit = true;
                    mine.where = fm;
                    mine.payload = pay;
                } else {
                    mine.where = fe < kNe ? fe : -1;
                }
            }
        }
    }
    return mine;
}

// Warp-cooperative probe with one 16-byte load per lane: the head of each
// lane's cell (head_n even, <= 8 slots: one 64-byte DRAM block) is read by
// head_n/2 adjacent lanes as one coalesced access, and every round's load is
// issued before the first decision, so a probe costs one DRAM round trip (the
// per-lane scans need two, and a random access that comes back to a row after
// it closed pays the row activation again). Per round one ballot finds, for
// each cell, the first 16-byte pair that ends the reference's linear scan (an
// empty slot or the matching check hash, cache.cpp:127-134), and the
// descriptor's lane reads the outcome from the deciding lane. A scan the head
// does not end continues in the cell's tail, lane by lane. Every lane of the
// warp must call it.
// Issue half of probe_warp16: every round's 16-byte head load for the warp's
// 32 cells (w[] holds them; lanes without a cell read ~0, which never ends a
// scan). Split from the resolve half so a kernel can keep several batches of
// loads in flight and do independent work (the next batch's hashes) while
// they are outstanding.
__device__ __forceinline__ void probe_warp16_issue(const CacheView& c, uint64_t cell, bool valid,
                                                   ulonglong2 (&w)[4]) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t lpc = c.head_n >> 1;      // lanes (pairs) per cell head
    const uint32_t cpr = 32u / lpc;          // cells per round
    const uint32_t rounds = (32u + cpr - 1u) / cpr;   // <= 4 for head_n <= 8
    const uint32_t g = lane / lpc, k = lane - g * lpc;
    // n_cells < 2^32 (mcg_cache_create), so a cell index fits one shuffle and
    // 0xffffffff can mark a lane without a cell.
    const uint32_t c32 = valid ? static_cast<uint32_t>(cell) : 0xffffffffu;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        w[r] = make_ulonglong2(~0ull, ~0ull);
        if (static_cast<uint32_t>(r) < rounds) {
            const uint32_t owner = static_cast<uint32_t>(r) * cpr + g;
            const uint32_t oc = __shfl_sync(kFull, c32, owner & 31u);
            if (g < cpr && owner < 32u && oc != 0xffffffffu) {
                w[r] = __ldcg(reinterpret_cast<const ulonglong2*>(head_words(c, oc)) + k);
            }
        }
    }
}

// Resolve half of probe_warp16 over the words probe_warp16_issue loaded.
__device__ __forceinline__ Probe probe_warp16_resolve(const CacheView& c, uint64_t cell, uint32_t check,
                                                      bool valid, const ulonglong2 (&w)[4]) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t lpc = c.head_n >> 1;
    const uint32_t cpr = 32u / lpc;
    const uint32_t rounds = (32u + cpr - 1u) / cpr;
    const uint32_t g = lane / lpc, k = lane - g * lpc;
    Probe mine{0u, -1, false};
    bool ended = false;
    const uint32_t my_round = lane / cpr, my_g = lane - my_round * cpr;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        if (static_cast<uint32_t>(r) >= rounds) break;
        const uint32_t chk = __shfl_sync(kFull, check, (static_cast<uint32_t>(r) * cpr + g) & 31u);
        const bool e0 = w[r].x == 0ull, m0 = static_cast<uint32_t>(w[r].x >> 32) == chk;
        const bool e1 = w[r].y == 0ull, m1 = static_cast<uint32_t>(w[r].y >> 32) == chk;
        const bool first0 = e0 || m0;
        const unsigned bal = __ballot_sync(kFull, (first0 || e1 || m1) && g < cpr);
        const bool hit = first0 ? (m0 && !e0) : (m1 && !e1);
        const uint32_t meta = ((2u * k + (first0 ? 0u : 1u)) << 1) | (hit ? 1u : 0u);
        const uint32_t pay = static_cast<uint32_t>(first0 ? w[r].x : w[r].y);
        uint32_t src = lane;
        bool found = false;
        if (my_round == static_cast<uint32_t>(r)) {
            const uint32_t bits = (bal >> (my_g * lpc)) & ((1u << lpc) - 1u);
            found = bits != 0u;
            src = my_g * lpc + (found ? static_cast<uint32_t>(__ffs(bits) - 1) : 0u);
        }
        const uint32_t m = __shfl_sync(kFull, meta, src);
        const uint32_t pl = __shfl_sync(kFull, pay, src);
        if (my_round == static_cast<uint32_t>(r) && found) {
            ended = true;
            mine.where = static_cast<int32_t>(m >> 1);
            mine.hit = (m & 1u) != 0u;
            if (mine.hit) mine.payload = pl;
        }
    }
    if (valid && !ended && c.n_entries > c.head_n) {
        const uint64_t* t = tail_words(c, cell);
        for (uint32_t j = 0; j < c.n_entries - c.head_n; ++j) {
            if (scan_word(__ldcg(t + j), static_cast<int32_t>(c.head_n + j), check, mine)) break;
        }
    }
    return mine;
}

// Resolve half through shared memory: the warp's loaded pairs are transposed
// through `tile` (4 rounds x 32 lanes x 16 B, this warp's slice) so that
// each lane then holds its own cell's head (head_n words) and scans it
// alone, branch-free: the first word that is empty or carries the check hash
// decides (cache.cpp:127-134). Same outcome as probe_warp16_resolve, with
// four shared-memory stores and head_n/2 loads instead of per-round ballots
// and shuffles. Every lane of the warp must call it.
__device__ __forceinline__ Probe probe_warp16_resolve_smem(const CacheView& c, uint64_t cell, uint32_t check,
                                                           bool valid, const ulonglong2 (&w)[4],
                                                           ulonglong2* tile) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t lpc = c.head_n >> 1;
    const uint32_t cpr = 32u / lpc;
    const uint32_t rounds = (32u + cpr - 1u) / cpr;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        if (static_cast<uint32_t>(r) < rounds) tile[r * 32 + lane] = w[r];
    }
    __syncwarp();
    const uint32_t my_round = lane / cpr, my_g = lane - my_round * cpr;
    const ulonglong2* mine_p = tile + my_round * 32u + my_g * lpc;
    uint32_t decisive = 0u, hitm = 0u;
    uint32_t pay[8];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        ulonglong2 q = make_ulonglong2(~0ull, ~0ull);
        if (static_cast<uint32_t>(k) < lpc) q = mine_p[k];
        const uint64_t x[2] = {q.x, q.y};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const bool in = static_cast<uint32_t>(k) < lpc;   // a slot of this cell's head
            const bool e = in && x[h] == 0ull;
            const bool m = in && static_cast<uint32_t>(x[h] >> 32) == check;
            decisive |= (e || m) ? (1u << (2 * k + h)) : 0u;
            hitm |= (m && !e) ? (1u << (2 * k + h)) : 0u;
            pay[2 * k + h] = static_cast<uint32_t>(x[h]);
        }
    }
    __syncwarp();   // the tile is reused by the next call
    Probe mine{0u, -1, false};
    if (decisive) {
        const int f = __ffs(decisive) - 1;
        mine.where = f;
        mine.hit = ((hitm >> f) & 1u) != 0u;
        uint32_t p = pay[0];
#pragma unroll
        for (int i = 1; i < 8; ++i) p = (f == i) ? pay[i] : p;
        if (mine.hit) mine.payload = p;
    } else if (valid && c.n_entries > c.head_n) {
        const uint64_t* t = tail_words(c, cell);
        for (uint32_t j = 0; j < c.n_entries - c.head_n; ++j) {
            if (scan_word(__ldcg(t + j), static_cast<int32_t>(c.head_n + j), check, mine)) break;
        }
    }
    return mine;
}

__device__ __forceinline__ Probe probe_warp16(const CacheView& c, uint64_t cell, uint32_t check,
                                              bool valid) {
    ulonglong2 w[4];
    probe_warp16_issue(c, cell, valid, w);
    return probe_warp16_resolve(c, cell, check, valid, w);
}

// Cooperative probe inside a lane group `grp` (the VM's material group,
// possibly a partial warp): the cells of the group's `leader` lanes are read
// by Ne/2 consecutive group lanes each, every round's load in flight before
// the first decision, as in probe_warp16. Falls back to per-lane scans by the
// leaders when the group is too small or has too many cells. Every lane of
// `grp` must call it; only leaders' results are meaningful.
__device__ __forceinline__ Probe probe_group16(const CacheView& c, uint64_t cell, uint32_t check,
                                              bool leader, unsigned grp) {
    const uint32_t lane = threadIdx.x & 31u;
    const unsigned L = __ballot_sync(grp, leader);
    const uint32_t nL = __popc(L), nW = __popc(grp);
    const uint32_t lpc = c.n_entries >> 1;
    const uint32_t cpr = lpc ? nW / lpc : 0u;
    const uint32_t rounds = cpr ? (nL + cpr - 1u) / cpr : 99u;
    if ((c.n_entries & 1u) != 0u || c.n_entries > c.head_n || cpr == 0u || rounds > 6u) {
        return leader ? probe_cell(c, cell, check) : Probe{0u, -1, false};
    }
    const unsigned below = (1u << lane) - 1u;
    const uint32_t rank = __popc(grp & below);
    const uint32_t g = rank / lpc, k = rank - g * lpc;
    ulonglong2 w[6];
#pragma unroll
    for (int r = 0; r < 6; ++r) {
        w[r] = make_ulonglong2(~0ull, ~0ull);
        if (static_cast<uint32_t>(r) < rounds) {
            const uint32_t j = static_cast<uint32_t>(r) * cpr + g;
            const bool work = g < cpr && j < nL;
            const uint32_t owner = work ? __fns(L, 0u, static_cast<int>(j) + 1) : lane;
            const uint64_t oc = __shfl_sync(grp, cell, owner);
            if (work) w[r] = __ldcg(reinterpret_cast<const ulonglong2*>(head_words(c, oc)) + k);
        }
    }
    Probe mine{0u, -1, false};
    const uint32_t jm = __popc(L & below);   // my ordinal among the leaders
    const uint32_t my_round = jm / cpr, gm = jm - my_round * cpr;
    unsigned range = 0u;
    if (leader) {
        const uint32_t lo = __fns(grp, 0u, static_cast<int>(gm * lpc) + 1);
        const uint32_t hi = __fns(grp, 0u, static_cast<int>(gm * lpc + lpc));
        const unsigned upto = hi >= 31u ? 0xffffffffu : ((2u << hi) - 1u);
        range = grp & upto & ~((1u << lo) - 1u);
    }
#pragma unroll
    for (int r = 0; r < 6; ++r) {
        if (static_cast<uint32_t>(r) >= rounds) break;
        const uint32_t j = static_cast<uint32_t>(r) * cpr + g;
        const bool work = g < cpr && j < nL;
        const uint32_t owner = work ? __fns(L, 0u, static_cast<int>(j) + 1) : lane;
        const uint32_t chk = __shfl_sync(grp, check, owner);
        const bool e0 = w[r].x == 0ull, m0 = static_cast<uint32_t>(w[r].x >> 32) == chk;
        const bool e1 = w[r].y == 0ull, m1 = static_cast<uint32_t>(w[r].y >> 32) == chk;
        const bool first0 = e0 || m0;
        const unsigned bal = __ballot_sync(grp, work && (first0 || e1 || m1));
        const bool hit = first0 ? (m0 && !e0) : (m1 && !e1);
        const uint32_t meta = ((2u * k + (first0 ? 0u : 1u)) << 1) | (hit ? 1u : 0u);
        const uint32_t pay = static_cast<uint32_t>(first0 ? w[r].x : w[r].y);
        uint32_t src = lane;
        bool found = false;
        if (leader && my_round == static_cast<uint32_t>(r)) {
            const unsigned bits = bal & range;
            found = bits != 0u;
            if (found) src = static_cast<uint32_t>(__ffs(bits) - 1);
        }
        const uint32_t mm = __shfl_sync(grp, meta, src);
        const uint32_t pl = __shfl_sync(grp, pay, src);
        if (leader && my_round == static_cast<uint32_t>(r)) {
            if (found) {
                mine.where = static_cast<int32_t>(mm >> 1);
                mine.hit = (mm & 1u) != 0u;
                if (mine.hit) mine.payload = pl;
            } else {
                mine.where = -1;
            }
        }
    }
    return mine;
}

// The warp's probes (batch lookups/updates, trace replay): the cooperative
// one-round-trip scan with the shared-memory resolve where the cell shape
// allows it (Ne even, head <= 8 slots), else the per-lane scan. `tile` is
// this warp's 128 ulonglong2 of shared memory. Warp-collective: every lane of
// the warp calls it (invalid lanes with valid = false).
__device__ __forceinline__ Probe probe_lanes_smem(const CacheView& c, uint64_t cell, uint32_t check,
                                                  bool valid, ulonglong2* tile) {
    if ((c.head_n & 1u) == 0u && c.head_n >= 2u && c.head_n <= 8u) {
        ulonglong2 w[4];
        probe_warp16_issue(c, cell, valid, w);
        return probe_warp16_resolve_smem(c, cell, check, valid, w, tile);
    }
    return valid ? probe_cell(c, cell, check) : Probe{0u, -1, false};
}

// CAS from zero; across devices (a striped table, peer memory over NVLink)
// only system-scope atomics are atomic with respect to the other GPUs.
__device__ __forceinline__ unsigned long long cas_slot(const CacheView& c, uint64_t* word,
                                                       unsigned long long packed) {
    unsigned long long* p = reinterpret_cast<unsigned long long*>(word);
    return c.world > 1u ? atomicCAS_system(p, 0ull, packed) : atomicCAS(p, 0ull, packed);
}

// update()'s insert (cache.cpp:94-119) from the scan's result: `where` is the
// first empty slot the probe saw (slots before it were occupied by other
// keys). The probe may have run long before the store (the VM probes at
// CacheLookup and stores at CacheStore, after the subtree), so a failed CAS
// continues the scan as update() would if it ran now: the winner's word
// holds our check hash -> AlreadyPresent; else the next slots are scanned
// (a match -> AlreadyPresent, the first empty one gets update()'s single
// CAS, whose failure is LostRace), and a full cell is CellFull. Slots before `where`
// never change (write-once), so this equals a full rescan at store time.
// Returns MCG_INSERT_*; *slot_out = the slot the outcome refers to (or -1).
__device__ __forceinline__ int insert_at(const CacheView& c, uint64_t cell, int32_t where,
                                         uint32_t check, uint32_t payload, int32_t* slot_out = nullptr) {
    if (slot_out) *slot_out = where;
    if (where < 0) return MCG_INSERT_CELL_FULL;
    const unsigned long long packed = (static_cast<unsigned long long>(check) << 32) | payload;
    unsigned long long prev = cas_slot(c, slot_ptr(c, cell, static_cast<uint32_t>(where)), packed);
    if (prev == 0ull) return MCG_INSERT_WON;
    if (static_cast<uint32_t>(prev >> 32) == check) return MCG_INSERT_ALREADY_PRESENT;
    for (uint32_t e = static_cast<uint32_t>(where) + 1u; e < c.n_entries; ++e) {
        if (slot_out) *slot_out = static_cast<int32_t>(e);
        uint64_t* w = slot_ptr(c, cell, e);
        const unsigned long long cur = *reinterpret_cast<volatile unsigned long long*>(w);
        if (static_cast<uint32_t>(cur >> 32) == check) return MCG_INSERT_ALREADY_PRESENT;
        if (cur == 0ull) {
            return cas_slot(c, w, packed) == 0ull ? MCG_INSERT_WON : MCG_INSERT_LOST_RACE;
        }
    }
    if (slot_out) *slot_out = -1;
    return MCG_INSERT_CELL_FULL;
}

// ---------------------------------------------------------------------------
// Scene view (device pointers; include/mcg.h layouts)
// ---------------------------------------------------------------------------
#ifndef MCG_SHADOW_WIDTH
#define MCG_SHADOW_WIDTH 4
#endif
constexpr int kShadowWidth = MCG_SHADOW_WIDTH;   // entries per node of the shadow tree
#ifndef MCG_CLOSEST_WIDTH
#define MCG_CLOSEST_WIDTH 4
#endif
constexpr int kClosestWidth = MCG_CLOSEST_WIDTH; // entries per node of the collapsed reference tree

struct SceneView {
    const float4* prim_geom;      // 3 float4 per prim
    const float2* prim_uv;        // 3 float2 per prim
    const uint32_t* prim_info;
    const float4* nodes;          // 2 float4 per BVH node (the reference tree, own boxes)
    const float4* pairs;          // 4 float4 per internal node: both children's records
    const float4* quads;          // 2 * kClosestWidth float4 per node (collapsed reference tree)
    int32_t root_a, root_b;       // root entry into `quads`: (0, -1) or a leaf (~first, count)
    const float4* squads;         // kShadowWidth-wide SAH tree over the reference's leaves (any-hit only)
    const float4* quads_soa;      // the 4-wide trees transposed: 8 float4 rows per node
    const float4* squads_soa;
    int32_t sroot_a, sroot_b;     // root entry into `squads`
    uint32_t n_nodes;
    const mcg_point_light* plights;
    uint32_t n_plights;
    const mcg_rect_light* rlights;
    uint32_t n_rlights;
    const mcg_program* programs;
    uint32_t n_programs;
    const mcg_insn* code;
    const mcg_const* consts;
    const mcg_noise* noise;
    const mcg_ramp* ramps;
    const mcg_ramp_stop* stops;
    const mcg_texture* textures;
    const float4* texels;
    uint32_t n_code;              // instruction words of all programs (shared-memory staging)
    float env[3];
    // Per program, its first kAhead cache points in bracket order: (node_idx,
    // flags | kAheadValid) -- what the look-ahead probe needs to build their
    // descriptors before the material sort (mcg_render.cu, k_lookahead).
    const uint2* ahead_cp;
};

// Cache points per material probed ahead of the shade (look_ahead, in the
// trace kernels); their results travel in the path's ray record: a flags
// word (bit c: cache point c hit; bit 8 + c: its cell was full without the
// key) and one payload word per cache point.
constexpr uint32_t kAhead = 8;
constexpr uint32_t kAheadValid = 0x100u;
constexpr uint32_t kAheadFull = 8u;   // flags shift of the cell-full bits

struct Ahead {
    uint32_t flags;
    const uint32_t* pay;   // kAhead payload words (in the path's record)
    bool on;
};

// Per-lane shading input (ShadingPoint, geom.hpp:49-56).
struct ShadeIn {
    float px, py, pz, nx, ny, nz, ix, iy, iz, u, v, g1x, g1y, g2x, g2y;
};

struct VmCounters {
    uint32_t instrs = 0, lookups = 0, hits = 0, stores = 0, won = 0, full = 0, tex = 0;
};

// Sink for deterministic-mode stores: (cell, pixel-order key) -> (check, payload).
struct StoreQueue {
    unsigned long long* keys;
    unsigned long long* vals;
    unsigned int* count;
    unsigned int capacity;
};

// Value stack in shared memory: three planes [slot][threads of the block];
// slot numbers are compile-time (mcg_insn.sp), so a warp always touches one
// row and the accesses are bank-conflict free.
struct Stack {
    float* x;
    float* y;
    float* z;
    int stride;
    int tid;
    int limit;   // the program's max_stack slots (checked builds)
    __device__ __forceinline__ void put(int s, float a, float b, float c, bool scalar) const {
        MCG_CHECK(s >= 0 && s < limit);
        x[s * stride + tid] = a;
        if (!scalar) {
            y[s * stride + tid] = b;
            z[s * stride + tid] = c;
        }
    }
    __device__ __forceinline__ float3 get(int s, bool scalar) const {
        MCG_CHECK(s >= 0 && s < limit);
        const float a = x[s * stride + tid];
        if (scalar) return make_float3(a, a, a);
        return make_float3(a, y[s * stride + tid], z[s * stride + tid]);
    }
    __device__ __forceinline__ float sx(int s) const { return x[s * stride + tid]; }
};

__device__ __forceinline__ float luminance(float3 c) {  // Value::as_scalar, value.hpp:36-38
    return 0.2126f * c.x + 0.7152f * c.y + 0.0722f * c.z;
}

__device__ __forceinline__ float bin_op(uint8_t op, float x, float y, float t) {
    switch (op) {
        case MCG_OP_ADD: return x + y;
        case MCG_OP_SUB: return x - y;
        case MCG_OP_MUL: return x * y;
        case MCG_OP_DIV: return y == 0.0f ? 0.0f : x / y;  // value.hpp:106-108
        case MCG_OP_MIX: return x * (1.0f - t) + y * t;    // value.hpp:110-113
        default: return power(x, y);                        // value.hpp:132-137
    }
}

struct VmResult {
    float3 value;
    bool scalar;
};

// Interprets material `slot` for every lane of `grp` (a set of lanes of this
// warp that all run the same program). The program counter is warp-uniform:
// the instruction word is one broadcast 16-byte load and the opcode switch
// never diverges. A lookup hit does not branch away: the lane parks until the
// bracket's resume point while the lanes that missed evaluate the subtree;
// when every lane of the group hits, the group jumps (skip_offset, Alg. 2).
//
// kDeferred: deterministic mode -- lookups read the epoch-start table and
// stores are queued with an order key (applied later, lowest key first);
// otherwise stores CAS immediately (concurrent mode).
#ifndef MCG_VM_REPROBE
#define MCG_VM_REPROBE 1   // concurrent mode: a look-ahead miss probes again at CacheLookup
#endif
template <bool kDeferred, bool kSmemCode = false>
// MCG_VM_PREFETCH=1 (experiment, off): fetch the next instruction word
// while the current one executes; neutral (636.6-637.7 vs 636.4-638.3 ms per
// bench render): the 16-byte words are L1 hits and not the VM's bound.
#ifndef MCG_VM_PREFETCH
#define MCG_VM_PREFETCH 0
#endif
__device__ __forceinline__ VmResult run_program(const SceneView& S, const CacheView& C,
                                                bool cache_on, int mip_offset, uint32_t slot,
                                                const ShadeIn& sp, unsigned grp, const Stack& st,
                                                const uint8_t* perm, uint32_t order_key,
                                                const StoreQueue& q, VmCounters& cnt,
                                                const Ahead& ah = Ahead{}, const uint4* s_code = nullptr,
                                                uint32_t s_code_base = 0) {
    const mcg_program prog = S.programs[slot];
    // kSmemCode: the program's words staged in shared memory by the calling
    // kernel from word s_code_base on (one 16-byte broadcast LDS per
    // dispatch); else L1-cached global loads
    const uint4* code = kSmemCode ? s_code + (prog.code_offset - s_code_base)
                                  : reinterpret_cast<const uint4*>(S.code) + prog.code_offset;
    const unsigned lane = threadIdx.x & 31u;
    bool parked = false;
    int resume = -1;
    uint32_t p_check = 0;
    int32_t p_where = -1;
    unsigned long long p_cell = 0;
    VmResult out{make_float3(0.0f, 0.0f, 0.0f), true};
#if MCG_VM_PREFETCH
    // the next word is fetched while this one executes (the upload pads the
    // code buffer by one word, so pc + 1 is always readable); a group skip
    // refetches at its target
    uint4 w_next = __ldg(code);
#endif
    for (int pc = 0;; ++pc) {
        if (pc == resume) {
            parked = false;
            resume = -1;
        }
#if MCG_VM_PREFETCH
        const uint4 w = w_next;
        w_next = __ldg(code + pc + 1);
#else
        MCG_CHECK(static_cast<uint32_t>(pc) < prog.code_len);
        const uint4 w = kSmemCode ? code[pc] : __ldg(code + pc);
#endif
        const uint8_t op = static_cast<uint8_t>(w.x & 0xffu);
        const uint8_t flags = static_cast<uint8_t>((w.x >> 8) & 0xffu);
        const int d = static_cast<int>((w.x >> 16) & 0xffu);
        const uint8_t tags = static_cast<uint8_t>(w.x >> 24);
        const uint32_t arg = w.y;
        const bool act = !parked;
        cnt.instrs += act ? 1u : 0u;
        const bool ta = tags & MCG_T_A, tb = tags & MCG_T_B, tc = tags & MCG_T_C,
                   tr = tags & MCG_T_R;
        switch (op) {
            case MCG_OP_PUSH_CONST:
                if (act) {
                    const float4 c = __ldg(reinterpret_cast<const float4*>(S.consts + arg));
                    st.put(d, c.x, c.y, c.z, tr);
                }
                break;
            case MCG_OP_LOAD_UV:
                if (act) {
                    const unsigned ch = (flags >> MCG_F_UV_SHIFT) & 3u;
                    if (ch == 0) st.put(d, sp.u, sp.v, 0.0f, false);
                    else st.put(d, ch == 1 ? sp.u : sp.v, 0.0f, 0.0f, true);
                }
                break;
            case MCG_OP_LOAD_POSITION:
                if (act) st.put(d, sp.px, sp.py, sp.pz, false);
                break;
            case MCG_OP_LOAD_NORMAL:
                if (act) st.put(d, sp.nx, sp.ny, sp.nz, false);
                break;
            case MCG_OP_LOAD_INCOMING:
                if (act) st.put(d, sp.ix, sp.iy, sp.iz, false);
                break;
            case MCG_OP_TEX_SAMPLE:
                if (act) {
                    const float3 c = bilinear(S.textures[arg], S.texels, sp.u, sp.v,
                                              (flags & MCG_F_WRAP_CLAMP) != 0);
                    st.put(d, c.x, c.y, c.z, false);
                    ++cnt.tex;
                }
                break;
            case MCG_OP_CHECKER:
                if (act) st.put(d, checker(__uint_as_float(w.w), sp.u, sp.v), 0.0f, 0.0f, true);
                break;
            case MCG_OP_NOISE:
                if (act) {
                    const float4 nz = __ldg(reinterpret_cast<const float4*>(S.noise + arg));
                    const mcg_noise p{__float_as_int(nz.x), nz.y, nz.z, nz.w};
                    st.put(d, fbm2(p, sp.u, sp.v, perm), 0.0f, 0.0f, true);
                }
                break;
            case MCG_OP_ADD: case MCG_OP_SUB: case MCG_OP_MUL: case MCG_OP_DIV: case MCG_OP_POWER:
                if (act) {
                    if (ta && tb) {
                        st.put(d - 2, bin_op(op, st.sx(d - 2), st.sx(d - 1), 0.0f), 0.0f, 0.0f, true);
                    } else {
                        const float3 a = st.get(d - 2, ta), b = st.get(d - 1, tb);
                        st.put(d - 2, bin_op(op, a.x, b.x, 0.0f), bin_op(op, a.y, b.y, 0.0f),
                               bin_op(op, a.z, b.z, 0.0f), false);
                    }
                }
                break;
            case MCG_OP_MIX:
                if (act) {
                    const float t = tc ? st.sx(d - 1) : luminance(st.get(d - 1, false));
                    if (ta && tb) {
                        st.put(d - 3, bin_op(MCG_OP_MIX, st.sx(d - 3), st.sx(d - 2), t), 0.0f, 0.0f, true);
                    } else {
                        const float3 a = st.get(d - 3, ta), b = st.get(d - 2, tb);
                        st.put(d - 3, bin_op(MCG_OP_MIX, a.x, b.x, t), bin_op(MCG_OP_MIX, a.y, b.y, t),
                               bin_op(MCG_OP_MIX, a.z, b.z, t), false);
                    }
                }
                break;
            case MCG_OP_CLAMP:
                if (act) {
                    const float3 a = st.get(d - 1, ta);
                    st.put(d - 1, fminf(fmaxf(a.x, 0.0f), 1.0f), fminf(fmaxf(a.y, 0.0f), 1.0f),
                           fminf(fmaxf(a.z, 0.0f), 1.0f), ta);
                }
                break;
            case MCG_OP_SIN_WAVE:
                if (act) {
                    if (ta) {
                        st.put(d - 1, sin_wave(st.sx(d - 1)), 0.0f, 0.0f, true);
                    } else {
                        const float3 a = st.get(d - 1, false);
                        st.put(d - 1, sin_wave(a.x), sin_wave(a.y), sin_wave(a.z), false);
                    }
                }
                break;
            case MCG_OP_DOT:  // value.hpp:119-123
                if (act) {
                    const float3 a = st.get(d - 2, ta), b = st.get(d - 1, tb);
                    st.put(d - 2, a.x * b.x + a.y * b.y + a.z * b.z, 0.0f, 0.0f, true);
                }
                break;
            case MCG_OP_RAMP:  // value.hpp:141-156
                if (act) {
                    const float t = ta ? st.sx(d - 1) : luminance(st.get(d - 1, false));
                    const mcg_ramp rp = S.ramps[arg];
                    const float4* s4 = reinterpret_cast<const float4*>(S.stops + rp.first);
                    float3 c = make_float3(0.0f, 0.0f, 0.0f);
                    if (rp.count > 0) {
                        const float4 first = __ldg(s4), last = __ldg(s4 + rp.count - 1);
                        if (t <= first.x) {
                            c = make_float3(first.y, first.z, first.w);
                        } else if (t >= last.x) {
                            c = make_float3(last.y, last.z, last.w);
                        } else {
                            c = make_float3(last.y, last.z, last.w);
                            float4 lo = first;
                            for (uint32_t i = 1; i < rp.count; ++i) {
                                const float4 hi = __ldg(s4 + i);
                                if (t <= hi.x) {
                                    const float span = hi.x - lo.x;
                                    const float wt = span > 0.0f ? (t - lo.x) / span : 0.0f;
                                    const float u = 1.0f - wt;
                                    c = make_float3(lo.y * u + hi.y * wt, lo.z * u + hi.z * wt,
                                                    lo.w * u + hi.w * wt);
                                    break;
                                }
                                lo = hi;
                            }
                        }
                    }
                    st.put(d - 1, c.x, c.y, c.z, false);
                }
                break;
            case MCG_OP_BSDF_DIFFUSE:
                if (act) {
                    const float3 a = st.get(d - 1, ta);
                    st.put(d - 1, a.x, a.y, a.z, false);
                }
                break;
            case MCG_OP_CACHE_LOOKUP: {  // stackvm.cpp:328-349
                if (!cache_on) break;
                // Brackets never nest, so every lane of the group is active here.
                // Cache points probed ahead of the shade (k_lookahead) take
                // that probe's result: the descriptor (and its hash, for the
                // store) is only built when a lane of the group missed.
                const uint32_t bi = w.z & 0xffffu;
                const bool ahead = ah.on && bi < kAhead;
                Probe pr{0u, -1, false};
                if (ahead) {
                    // (no slot hint: a miss in a cell with room probes again
                    // below -- concurrent mode -- or is queued -- deterministic)
                    pr.hit = ((ah.flags >> bi) & 1u) != 0u;
                    if (pr.hit) pr.payload = __ldg(ah.pay + bi);
                    pr.where = ((ah.flags >> (kAheadFull + bi)) & 1u) ? -1 : 0;
                }
                // (No lane needs the descriptor when every lane hit, or --
                // concurrent mode -- every lane's look-ahead found its cell
                // full: no probe and no insert can follow.)
                if (!ahead || C.trace ||
                    !__all_sync(grp, pr.hit || (!kDeferred && MCG_VM_REPROBE && pr.where < 0))) {
                    Desc desc{prog.material_id, arg, 0u, 0u, 0u};
                    if (flags & MCG_F_USES_UV) {
                        desc.mip = mip_level(sp.g1x, sp.g1y, sp.g2x, sp.g2y, mip_offset);
                        desc.tx = texel_index(sp.u, desc.mip);
                        desc.ty = texel_index(sp.v, desc.mip);
                    }
                    uint64_t h;
                    hash_desc(desc, h, p_check);
                    const uint64_t cell = fast_mod(h, C.n_cells, C.magic);
                    p_cell = cell;
                    // Probe now: without a look-ahead result, or (concurrent
                    // mode) again for a look-ahead miss -- a store that landed
                    // since then is a hit, as it would be for the reference's
                    // lookup at this point. (Deterministic mode reads the
                    // epoch-start table, which the look-ahead already saw.)
                    // (A look-ahead that found the cell full without the key is
                    // final: slots are write-once, so the key can never enter
                    // that cell -- no second probe.)
                    const bool probe_now = !ahead || (MCG_VM_REPROBE && !kDeferred && !pr.hit && pr.where >= 0);
                    const unsigned pm = __ballot_sync(grp, probe_now);
                    if (probe_now) {
                        // Lanes asking for the same (cell, check) share one probe.
                        const unsigned long long key = (cell << 32) ^ p_check;
                        const unsigned peers = __match_any_sync(pm, key);
                        const int leader = __ffs(peers) - 1;
#ifdef MCG_VM_GROUP_PROBE
                        // cooperative scan by the group (measured slower in the VM:
                        // 115 vs 96 registers, and few leaders per warp after the
                        // Morton sort -- profiles/README.md)
                        pr = probe_group16(C, p_cell, p_check, static_cast<int>(lane) == leader, pm);
#else
                        Probe np{0u, -1, false};
                        if (static_cast<int>(lane) == leader) np = probe_cell_t<MCG_VM_FIRST_PAIRS>(C, p_cell, p_check);
                        pr = np;
#endif
                        pr.payload = __shfl_sync(peers, pr.payload, leader);
                        pr.where = __shfl_sync(peers, pr.where, leader);
                        pr.hit = __shfl_sync(peers, static_cast<int>(pr.hit), leader) != 0;
                    }
                    if (C.trace) {
                        // descriptor log (SURVEY §8d trace replay): warp-aggregated append
                        const int ldr = __ffs(grp) - 1;
                        unsigned long long at = 0;
                        if (static_cast<int>(lane) == ldr) at = atomicAdd(C.trace_count, __popc(grp));
                        at = __shfl_sync(grp, at, ldr) + __popc(grp & ((1u << lane) - 1u));
                        if (at < C.trace_cap) {
                            uint32_t* t = C.trace + 5 * at;
                            t[0] = desc.mat;
                            t[1] = desc.node;
                            t[2] = desc.mip;
                            t[3] = desc.tx;
                            t[4] = desc.ty;
                        }
                    }
                }
                ++cnt.lookups;
                p_where = pr.where;
                if (pr.hit) {
                    const float3 v = decode_rgbe(pr.payload);
                    if (flags & MCG_F_SCALAR_RESULT) st.put(d, v.x, 0.0f, 0.0f, true);
                    else st.put(d, v.x, v.y, v.z, false);
                    ++cnt.hits;
                    parked = true;
                }
                const int skip = static_cast<int>(w.w);
                if (__all_sync(grp, pr.hit)) {
                    parked = false;
                    pc += skip;  // the whole group skips the subtree
#if MCG_VM_PREFETCH
                    w_next = __ldg(code + pc + 1);
#endif
                } else {
                    resume = pc + 1 + skip;
                }
                break;
            }
            case MCG_OP_CACHE_STORE: {  // stackvm.cpp:350-357
                if (!cache_on) break;
                const unsigned m = __ballot_sync(grp, act);
                if (act) {
                    ++cnt.stores;
                    const float3 v = st.get(d - 1, ta);
                    // (a cell seen full takes no insert: no payload needed)
                    const uint32_t payload = (kDeferred || p_where >= 0) ? encode_rgbe(v.x, v.y, v.z) : 0u;
                    if (kDeferred) {
                        const unsigned rank = __popc(m & ((1u << lane) - 1u));
                        const int ldr = __ffs(m) - 1;
                        unsigned base = 0;
                        if (static_cast<int>(lane) == ldr) base = atomicAdd(q.count, __popc(m));
                        base = __shfl_sync(m, base, ldr);
                        const unsigned pos = base + rank;
                        if (pos < q.capacity) {
                            q.keys[pos] = (p_cell << 32) |
                                          static_cast<unsigned long long>(order_key | ((w.z >> 16) & 0xffu));
                            q.vals[pos] = (static_cast<unsigned long long>(p_check) << 32) | payload;
                        }
                    } else {
                        // One CAS per distinct (cell, check) in the warp; the
                        // others saw the same empty slot and now find it taken
                        // by their own key (AlreadyPresent).
                        // The group's CAS carries the value of a lane picked by
                        // a hash of its path key, not the lowest lane: lanes sit
                        // in Morton order, so "lowest" would always store the
                        // value at one corner of the texel (a biased first insert).
                        const unsigned long long key = (p_cell << 32) ^ p_check;
                        const unsigned peers = __match_any_sync(m, key);
                        const uint32_t rk = (order_key >> 6) * 0x9E3779B1u;
                        const uint32_t rmin = __reduce_min_sync(peers, rk);
                        const int leader = __ffs(__ballot_sync(peers, rk == rmin) & peers) - 1;
                        int res = MCG_INSERT_ALREADY_PRESENT;
                        if (static_cast<int>(lane) == leader) {
                            int32_t at = -1;
                            res = insert_at(C, p_cell, p_where, p_check, payload, &at);
                            if (C.ilog && res == MCG_INSERT_WON) {
                                // the descriptor again (CacheStore carries the
                                // cache point's node and uv flag, stackvm.cpp:350-357)
                                uint32_t mip = 0, tx = 0, ty = 0;
                                if (flags & MCG_F_USES_UV) {
                                    mip = mip_level(sp.g1x, sp.g1y, sp.g2x, sp.g2y, mip_offset);
                                    tx = texel_index(sp.u, mip);
                                    ty = texel_index(sp.v, mip);
                                }
                                log_insert(C, prog.material_id, arg, mip, tx, ty, static_cast<uint32_t>(at), payload);
                            }
                        } else if (p_where < 0) {
                            res = MCG_INSERT_CELL_FULL;
                        }
                        cnt.won += res == MCG_INSERT_WON;
                        cnt.full += res == MCG_INSERT_CELL_FULL;
                    }
                }
                break;
            }
            case MCG_OP_END:
            default: {
                out.value = st.get(d - 1, ta);
                out.scalar = tr;
                return out;
            }
        }
    }
}

// Warp-aggregated counter update: one atomic per warp.
__device__ __forceinline__ void warp_add(unsigned long long* dst, uint32_t v) {
    const unsigned m = __activemask();
    const uint32_t s = __reduce_add_sync(m, v);
    if ((threadIdx.x & 31u) == static_cast<unsigned>(__ffs(m) - 1) && s) atomicAdd(dst, static_cast<unsigned long long>(s));
}

}  // namespace mcgd

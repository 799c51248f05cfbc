// Host-side device runtime state shared by the .cu translation units.
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <string>
#include <vector>

#include "host_internal.hpp"
#include "mcg_device.cuh"

namespace mcg {

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        fail(e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver ? MCG_ERR_NO_DEVICE
                                                                        : MCG_ERR_CUDA,
             std::string(what) + ": " + cudaGetErrorString(e));
    }
}

// Growable device buffer (capacity only grows; contents undefined after grow).
struct DevMem {
    void* p = nullptr;
    size_t bytes = 0;
    void ensure(size_t need) {
        if (need <= bytes) return;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        cuda_check(cudaMalloc(&p, need), "cudaMalloc");
        bytes = need;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
};

struct KernelAcc {
    uint64_t launches = 0;
    double ms = 0.0;
    double bytes = 0.0;
};

struct EventRec {
    std::string name;
    cudaEvent_t a, b;
    double bytes;
};

// Device copy of a prepared scene.
struct DeviceScene {
    std::vector<DevMem> bufs;
    mcgd::SceneView view{};
    uint32_t max_stack = 1;
    uint32_t max_cache_points = 0;
    float root_lo[3] = {0, 0, 0}, root_hi[3] = {0, 0, 0};   // scene bounds (BVH root)
    uint32_t max_stack4 = 1;   // worst-case LIFO stack of the 4-wide traversal
    uint32_t max_stack_s = 1;  // same for the shadow (SAH) tree
    std::vector<mcg_bvh_node> shadow_nodes;   // host copy of the shadow tree (mcg_shadow_tree)
    mcg_flat_scene cam{};   // camera/env fields only (no pointers used)
    bool loaded = false;
    void clear() {
        for (DevMem& m : bufs) m.release();
        bufs.clear();
        view = mcgd::SceneView{};
        loaded = false;
    }
    // A new upload reuses the device buffers (grown when too small):
    // cudaFree/cudaMalloc per upload cost tens to hundreds of ms.
    void reset() {
        view = mcgd::SceneView{};
        loaded = false;
    }
};

}  // namespace mcg

// Slots of a cell kept in the head array: one 64-byte DRAM block
// (mcg_device.cuh head_words); the rest go to the tail array.
inline uint32_t head_slots(uint32_t n_entries) { return n_entries > 8u ? 8u : n_entries; }

struct mcg_cache {
    mcg_ctx* ctx = nullptr;
    uint64_t n_cells = 0;         // logical cells (all stripes)
    uint32_t n_entries = 0;
    uint32_t head_n = 0;          // slots per cell in the head array (head_slots(n_entries))
    uint64_t magic = 0;
    uint64_t* slots = nullptr;    // this device's cells (all of them when world == 1)
    unsigned long long* counters = nullptr;  // lookups, hits, won, lost_full, lost_race
    // Striped shared table: this stripe holds cells c with
    // c % world == rank; `stripes` (device array) points at every stripe,
    // peers' through CUDA IPC / peer access over NVLink.
    uint32_t world = 1, rank = 0;
    uint64_t local_cells = 0;
    uint64_t** stripes = nullptr;
    std::vector<void*> ipc_opened;
    // descriptor trace of the lookups made through this table (mcg_cache_trace_*)
    uint32_t* trace = nullptr;
    unsigned long long* trace_count = nullptr;
    uint64_t trace_cap = 0;
    // won-insert log (mcg_cache_insert_log_*): 7 words per record
    uint32_t* ilog = nullptr;
    unsigned long long* ilog_count = nullptr;
    uint64_t ilog_cap = 0, ilog_alloc = 0;
    uint64_t local_words() const { return local_cells * n_entries; }   // slots held here (head + tail)
    uint64_t* tail() const { return n_entries > head_n ? slots + local_cells * head_n : nullptr; }
    mcgd::CacheView view() const {
        return {slots, tail(), n_cells, magic, n_entries, head_n, world, stripes, trace, trace_count, trace_cap,
                ilog_cap ? ilog : nullptr, ilog_count, ilog_cap};
    }
};

struct mcg_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    bool profile = false;
    uint64_t launches = 0;       // this library's kernels
    uint64_t library_sorts = 0;  // cub::DeviceRadixSort invocations
    std::map<std::string, mcg::KernelAcc> times;
    std::vector<mcg::EventRec> pending;
    std::vector<cudaEvent_t> event_pool;
    mcg::DeviceScene scene;
    mcg_cache* own_cache = nullptr;
    // second stream for work that overlaps the main one (shadow rays while
    // the continuation rays are traced), joined through the two events
    cudaStream_t aux = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    // further pass lanes (render passes in flight on several stream pairs):
    // their main and aux streams, fork/join events, path state and sort
    // scratch ([0] unused: lane 0 is stream/aux/ev_fork/ev_join/path_mem);
    // ev_lane[l] marks lane l's last accumulate, ev_lane[kMaxLanes] the
    // render's start and end
    static constexpr int kMaxLanes = 4;
    cudaStream_t lane_stream[kMaxLanes] = {}, lane_aux[kMaxLanes] = {};
    cudaEvent_t lane_fork[kMaxLanes] = {}, lane_join[kMaxLanes] = {};
    cudaEvent_t ev_lane[kMaxLanes + 1] = {};
    mcg::DevMem lane_cub[kMaxLanes], lane_path[kMaxLanes];
    // the shard's pixel list, device-resident across render calls with the
    // same (width, height, tile size, shard rank, count, mode)
    mcg::DevMem pix_mem;
    int64_t pix_key[6] = {-1, -1, -1, -1, -1, -1};
    uint32_t pix_n = 0;
    // scratch
    mcg::DevMem cub_temp, scratch_a, scratch_b, scratch_c, scratch_d, scratch_e;
    mcg::DevMem path_mem, queue_mem, stats_mem;
    // in-process multi-GPU (mcg_options.n_devices > 1): one single-device
    // context per further device, NCCL communicators over all of them
    // (created on the first multi-device render; distinct devices only)
    std::vector<mcg_ctx*> peers;
    std::vector<void*> nccl_comms;
    bool devices_distinct = true;
    mcg::DevMem build_mem;    // device BVH build scratch (mcg_build.cu)
    mcg::DevMem gather_tmp;   // device-copy gather (a device listed twice)
};

namespace mcg {

cudaEvent_t take_event(mcg_ctx* ctx);
void resolve_events(mcg_ctx* ctx);  // synchronizes on the pending events
void nccl_destroy(mcg_ctx* ctx);    // the multi-device context's communicators (mcg_render.cu)

// Brackets one kernel launch: counts it and, when profiling, records CUDA
// events on the context stream around it.
class LaunchScope {
public:
    LaunchScope(mcg_ctx* ctx, const char* name, double bytes, cudaStream_t stream = nullptr)
        : ctx_(ctx), name_(name), bytes_(bytes), stream_(stream ? stream : ctx->stream) {
        if (ctx_->profile) {
            a_ = take_event(ctx_);
            cudaEventRecord(a_, stream_);
        }
    }
    void done() {
        cuda_check(cudaGetLastError(), name_);
        ++ctx_->launches;
        if (ctx_->profile) {
            cudaEvent_t b = take_event(ctx_);
            cudaEventRecord(b, stream_);
            ctx_->pending.push_back({name_, a_, b, bytes_});
        }
    }

private:
    mcg_ctx* ctx_;
    const char* name_;
    double bytes_;
    cudaStream_t stream_;
    cudaEvent_t a_ = nullptr;
};

inline unsigned grid_for(size_t n, unsigned block) {
    return static_cast<unsigned>((n + block - 1) / block);
}

inline uint64_t mod_magic(uint64_t n) { return ~0ull / n; }

inline int bits_for(uint64_t v) {  // bits needed to hold values in [0, v]
    int b = 0;
    while (b < 64 && (v >> b) != 0) ++b;
    return b;
}

void sort_pairs_u64(mcg_ctx* ctx, const unsigned long long* keys_in, unsigned long long* keys_out,
                    const unsigned long long* vals_in, unsigned long long* vals_out, size_t n,
                    int end_bit);
void sort_pairs_u32(mcg_ctx* ctx, const uint32_t* keys_in, uint32_t* keys_out,
                    const uint32_t* vals_in, uint32_t* vals_out, size_t n, int end_bit,
                    cudaStream_t stream = nullptr, DevMem* temp = nullptr);

// The any-hit tree over the reference BVH's leaves (build_shadow_tree's
// binned SAH, collapsed to `width`-wide nodes), built on the device
// (mcg_build.cu).
std::vector<mcg_bvh_node> build_shadow_tree_device(mcg_ctx* ctx, const std::vector<mcg_bvh_node>& leaves,
                                                   int width, int32_t& root_a, int32_t& root_b);

// Applies sorted (cell << order_bits | order) -> (check << 32 | payload)
// records cell by cell in order (the deterministic-insert rule). Outcomes are
// optionally scattered back to index = order.
void apply_ordered(mcg_ctx* ctx, mcg_cache* cache, const unsigned long long* keys,
                   const unsigned long long* vals, size_t n, int order_bits, uint8_t* d_outcome,
                   uint64_t* d_slot, uint64_t* d_packed, unsigned long long* d_stats);

}  // namespace mcg

// Device build of the any-hit (shadow) hierarchy: the binned-SAH tree over
// the reference BVH's leaves that build_shadow_tree (mcg_runtime.cu) builds
// on the host, built on the GPU.
//
// Any hierarchy over the reference's leaves (same leaf boxes, same primitive
// ranges) answers Scene::occluded (scene.cpp:280-298) exactly as the
// reference's own tree does, so the device build only has to
// be a good tree; it is also the *same* tree as the host build: the same
// 32-bin SAH over leaf centroids, the same float/double arithmetic and the
// same tie rules, level by level:
//
//   k_sah_level   one block per node of the current level: node and centroid
//                 bounds (block reduction), 3 x 32 bins (shared-memory
//                 atomics on order-preserving integer images of the floats,
//                 so min/max are exact), the host's prefix/suffix sweep by one
//                 thread, then the node's leaf indices permuted exactly as
//                 the host's std::partition permutes them (computed in
//                 parallel) into the next level's array
//   k_collapse    the binary tree to `width`-wide nodes, top-down, a node per
//                 thread: open the largest-area internal entry until the node
//                 holds `width` entries (the host's rule), allocate child
//                 nodes with an atomic counter
//
// Only node numbering differs from the host (breadth-first here, depth-first
// there; traversal does not depend on it). Leaf order inside a node's range
// matters where every leaf centroid coincides (no SAH split: the host takes
// an index median), so the partition reproduces libstdc++'s permutation.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "mcg_ctx.cuh"

namespace {

constexpr int kBins = 32;
constexpr int kBuildBlock = 256;

struct SahTask {
    int32_t node, first, count, pad;
};

struct BinNode {
    float lo[3], hi[3];
    int32_t l, r, leaf, pad;
};

// Order-preserving integer image of a float (min/max with integer atomics).
__device__ __forceinline__ int ord(float f) {
    const int i = __float_as_int(f);
    return i >= 0 ? i : i ^ 0x7fffffff;
}
__device__ __forceinline__ float unord(int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7fffffff); }

__device__ __forceinline__ float area3(const float* lo, const float* hi) {
    const float dx = hi[0] - lo[0], dy = hi[1] - lo[1], dz = hi[2] - lo[2];
    return dx * dy + dy * dz + dz * dx;
}

__device__ __forceinline__ float cen(const mcg_bvh_node& L, int a) { return 0.5f * (L.lo[a] + L.hi[a]); }

__device__ __forceinline__ int bin_of(float c, float clo, float ext) {
    int b = static_cast<int>((c - clo) / ext * kBins);
    return min(max(b, 0), kBins - 1);
}

__global__ void __launch_bounds__(kBuildBlock) k_sah_level(const mcg_bvh_node* __restrict__ leaves,
                                                           const int32_t* __restrict__ idx_in,
                                                           int32_t* __restrict__ idx_out,
                                                           const SahTask* __restrict__ tasks,
                                                           BinNode* __restrict__ bn, SahTask* __restrict__ next,
                                                           int32_t* counters, int32_t* __restrict__ scratch) {
    __shared__ int s_lo[3], s_hi[3], s_clo[3], s_chi[3];
    __shared__ int s_cnt[3][kBins], s_blo[3][kBins][3], s_bhi[3][kBins][3];
    __shared__ int s_axis, s_bin, s_left, s_tl;
    __shared__ int s_scan[kBuildBlock / 32], s_scan2[kBuildBlock / 32];
    const SahTask t = tasks[blockIdx.x];
    const int tid = threadIdx.x;
    if (tid < 3) {
        s_lo[tid] = s_clo[tid] = ord(__int_as_float(0x7f800000));
        s_hi[tid] = s_chi[tid] = ord(__int_as_float(0xff800000));
    }
    for (int k = tid; k < 3 * kBins; k += blockDim.x) {
        const int a = k / kBins, b = k % kBins;
        s_cnt[a][b] = 0;
        for (int c = 0; c < 3; ++c) {
            s_blo[a][b][c] = ord(__int_as_float(0x7f800000));
            s_bhi[a][b][c] = ord(__int_as_float(0xff800000));
        }
    }
    __syncthreads();
    // node bounds and centroid bounds
    {
        float lo[3], hi[3], clo[3], chi[3];
        for (int a = 0; a < 3; ++a) {
            lo[a] = clo[a] = __int_as_float(0x7f800000);
            hi[a] = chi[a] = __int_as_float(0xff800000);
        }
        for (int k = t.first + tid; k < t.first + t.count; k += blockDim.x) {
            const mcg_bvh_node L = leaves[idx_in[k]];
            for (int a = 0; a < 3; ++a) {
                lo[a] = fminf(lo[a], L.lo[a]);
                hi[a] = fmaxf(hi[a], L.hi[a]);
                clo[a] = fminf(clo[a], cen(L, a));
                chi[a] = fmaxf(chi[a], cen(L, a));
            }
        }
        for (int a = 0; a < 3; ++a) {
            atomicMin(&s_lo[a], ord(lo[a]));
            atomicMax(&s_hi[a], ord(hi[a]));
            atomicMin(&s_clo[a], ord(clo[a]));
            atomicMax(&s_chi[a], ord(chi[a]));
        }
    }
    __syncthreads();
    if (t.count == 1) {
        if (tid == 0) {
            BinNode nd;
            for (int a = 0; a < 3; ++a) {
                nd.lo[a] = unord(s_lo[a]);
                nd.hi[a] = unord(s_hi[a]);
            }
            nd.l = nd.r = -1;
            nd.leaf = idx_in[t.first];
            nd.pad = 0;
            bn[t.node] = nd;
        }
        return;
    }
    float clo[3], ext[3];
    for (int a = 0; a < 3; ++a) {
        clo[a] = unord(s_clo[a]);
        ext[a] = unord(s_chi[a]) - clo[a];
    }
    // 3 x 32 bins over the centroids
    for (int k = t.first + tid; k < t.first + t.count; k += blockDim.x) {
        const mcg_bvh_node L = leaves[idx_in[k]];
        for (int a = 0; a < 3; ++a) {
            if (!(ext[a] > 0.0f)) continue;
            const int b = bin_of(cen(L, a), clo[a], ext[a]);
            atomicAdd(&s_cnt[a][b], 1);
            for (int c = 0; c < 3; ++c) {
                atomicMin(&s_blo[a][b][c], ord(L.lo[c]));
                atomicMax(&s_bhi[a][b][c], ord(L.hi[c]));
            }
        }
    }
    __syncthreads();
    if (tid == 0) {
        // build_shadow_tree's sweep, operation for operation
        double best = __longlong_as_double(0x7ff0000000000000ll);
        int best_axis = -1, best_bin = 0;
        for (int a = 0; a < 3; ++a) {
            if (!(ext[a] > 0.0f)) continue;
            float rlo[kBins][3], rhi[kBins][3];
            int rcnt[kBins];
            float alo[3], ahi[3];
            int acnt = 0;
            for (int c = 0; c < 3; ++c) {
                alo[c] = __int_as_float(0x7f800000);
                ahi[c] = __int_as_float(0xff800000);
            }
            for (int b = kBins - 1; b >= 0; --b) {
                acnt += s_cnt[a][b];
                for (int c = 0; c < 3; ++c) {
                    alo[c] = fminf(alo[c], unord(s_blo[a][b][c]));
                    ahi[c] = fmaxf(ahi[c], unord(s_bhi[a][b][c]));
                    rlo[b][c] = alo[c];
                    rhi[b][c] = ahi[c];
                }
                rcnt[b] = acnt;
            }
            for (int c = 0; c < 3; ++c) {
                alo[c] = __int_as_float(0x7f800000);
                ahi[c] = __int_as_float(0xff800000);
            }
            acnt = 0;
            for (int b = 0; b < kBins - 1; ++b) {
                acnt += s_cnt[a][b];
                for (int c = 0; c < 3; ++c) {
                    alo[c] = fminf(alo[c], unord(s_blo[a][b][c]));
                    ahi[c] = fmaxf(ahi[c], unord(s_bhi[a][b][c]));
                }
                if (acnt == 0 || rcnt[b + 1] == 0) continue;
                const double cost = static_cast<double>(area3(alo, ahi)) * acnt +
                                    static_cast<double>(area3(rlo[b + 1], rhi[b + 1])) * rcnt[b + 1];
                if (cost < best) {
                    best = cost;
                    best_axis = a;
                    best_bin = b;
                }
            }
        }
        s_axis = best_axis;
        s_bin = best_bin;
        s_left = 0;
        s_tl = 0;
    }
    __syncthreads();
    const int axis = s_axis, bsplit = s_bin;
    // left count, then a stable partition (chunks of the block, warp scans)
    if (axis >= 0) {
        int mine = 0;
        for (int k = t.first + tid; k < t.first + t.count; k += blockDim.x) {
            mine += bin_of(cen(leaves[idx_in[k]], axis), clo[axis], ext[axis]) <= bsplit;
        }
        atomicAdd(&s_left, mine);
    }
    __syncthreads();
    int left = axis >= 0 ? s_left : 0;
    const bool split = axis >= 0 && left > 0 && left < t.count;
    if (!split) {
        left = t.count / 2;  // index median (build_shadow_tree's fallback)
        for (int k = t.first + tid; k < t.first + t.count; k += blockDim.x) idx_out[k] = idx_in[k];
    } else {
        // The permutation std::partition makes (libstdc++'s bidirectional
        // __partition, the host builder's call): with L = #true, the j-th
        // false of [0, L) from the left swaps with the j-th true of [L, n)
        // from the right; everything else stays. Computed in parallel:
        // copy, rank the misplaced elements (block scans), swap pairs.
        for (int k = t.first + tid; k < t.first + t.count; k += blockDim.x) idx_out[k] = idx_in[k];
        int tl = 0;   // trues in [0, L)
        for (int k = t.first + tid; k < t.first + left; k += blockDim.x) {
            tl += bin_of(cen(leaves[idx_in[k]], axis), clo[axis], ext[axis]) <= bsplit;
        }
        atomicAdd(&s_tl, tl);
        __syncthreads();
        const int m = left - s_tl;   // misplaced pairs
        const int lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
        int base_f = 0, base_t = 0;
        for (int c0 = t.first; c0 < t.first + t.count; c0 += blockDim.x) {
            const int k = c0 + tid;
            const bool valid = k < t.first + t.count;
            const bool p = valid && bin_of(cen(leaves[idx_in[k]], axis), clo[axis], ext[axis]) <= bsplit;
            const bool in_left = k - t.first < left;
            const bool fl = valid && in_left && !p, tr = valid && !in_left && p;
            const unsigned bf = __ballot_sync(0xffffffffu, fl), bt = __ballot_sync(0xffffffffu, tr);
            if (lane == 0) {
                s_scan[warp] = __popc(bf);
                s_scan2[warp] = __popc(bt);
            }
            __syncthreads();
            int bef_f = 0, bef_t = 0, tot_f = 0, tot_t = 0;
            for (int w = 0; w < nw; ++w) {
                if (w < warp) {
                    bef_f += s_scan[w];
                    bef_t += s_scan2[w];
                }
                tot_f += s_scan[w];
                tot_t += s_scan2[w];
            }
            const unsigned below = (1u << lane) - 1u;
            if (fl) scratch[t.first + base_f + bef_f + __popc(bf & below)] = k - t.first;
            if (tr) scratch[t.first + left + (m - 1 - (base_t + bef_t + __popc(bt & below)))] = k - t.first;
            base_f += tot_f;
            base_t += tot_t;
            __syncthreads();
        }
        for (int j = tid; j < m; j += blockDim.x) {
            const int a = scratch[t.first + j], b = scratch[t.first + left + j];
            idx_out[t.first + a] = idx_in[t.first + b];
            idx_out[t.first + b] = idx_in[t.first + a];
        }
    }
    if (tid == 0) {
        const int l = atomicAdd(&counters[1], 2);
        BinNode nd;
        for (int a = 0; a < 3; ++a) {
            nd.lo[a] = unord(s_lo[a]);
            nd.hi[a] = unord(s_hi[a]);
        }
        nd.l = l;
        nd.r = l + 1;
        nd.leaf = -1;
        nd.pad = 0;
        bn[t.node] = nd;
        const int at = atomicAdd(&counters[0], 2);
        next[at] = SahTask{l, t.first, left, 0};
        next[at + 1] = SahTask{l + 1, t.first + left, t.count - left, 0};
    }
}

// (binary node, output node) pairs of one level of the collapse.
struct CollapseTask {
    int32_t bnode, q;
};

__global__ void k_collapse(const BinNode* __restrict__ bn, const mcg_bvh_node* __restrict__ leaves,
                           const CollapseTask* __restrict__ tasks, int n_tasks, int width,
                           mcg_bvh_node* __restrict__ out, CollapseTask* __restrict__ next, int32_t* counters) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_tasks) return;
    const CollapseTask t = tasks[i];
    int32_t e[8];
    int n = 2;
    e[0] = bn[t.bnode].l;
    e[1] = bn[t.bnode].r;
    while (n < width) {
        int best = -1;
        float best_area = -1.0f;
        for (int k = 0; k < n; ++k) {
            const BinNode& b = bn[e[k]];
            if (b.leaf >= 0) continue;
            const float a = area3(b.lo, b.hi);
            if (a > best_area) {
                best_area = a;
                best = k;
            }
        }
        if (best < 0) break;
        const int32_t x2 = e[best];
        for (int k = n; k > best + 1; --k) e[k] = e[k - 1];
        e[best] = bn[x2].l;
        e[best + 1] = bn[x2].r;
        ++n;
    }
    for (int k = 0; k < n; ++k) {
        const BinNode& b = bn[e[k]];
        mcg_bvh_node rec;
        if (b.leaf >= 0) {
            rec = leaves[b.leaf];
        } else {
            for (int a = 0; a < 3; ++a) {
                rec.lo[a] = b.lo[a];
                rec.hi[a] = b.hi[a];
            }
            const int q2 = atomicAdd(&counters[1], 1);
            rec.a = q2;
            rec.b = -1;
            next[atomicAdd(&counters[0], 1)] = CollapseTask{e[k], q2};
        }
        out[static_cast<size_t>(width) * t.q + k] = rec;
    }
}

}  // namespace

namespace mcg {

std::vector<mcg_bvh_node> build_shadow_tree_device(mcg_ctx* ctx, const std::vector<mcg_bvh_node>& leaves,
                                                   int width, int32_t& root_a, int32_t& root_b) {
    std::vector<mcg_bvh_node> out;
    root_a = 0;
    root_b = 0;
    if (leaves.empty()) return out;
    if (leaves.size() == 1) {
        root_a = leaves[0].a;
        root_b = leaves[0].b;
        return out;
    }
    if (width < 2 || width > 8) fail(MCG_ERR_INVALID_ARGUMENT, "shadow tree width must be in [2, 8]");
    const int n = static_cast<int>(leaves.size());
    cudaStream_t s = ctx->stream;
    DevMem& m = ctx->build_mem;
    // leaves | idx x2 | tasks x2 | binary nodes | counters | output nodes | collapse tasks x2
    const size_t b_leaves = static_cast<size_t>(n) * sizeof(mcg_bvh_node);
    const size_t b_idx = static_cast<size_t>(n) * 4;
    const size_t b_tasks = static_cast<size_t>(2 * n) * sizeof(SahTask);
    const size_t b_bn = static_cast<size_t>(2 * n) * sizeof(BinNode);
    const size_t b_out = static_cast<size_t>(n) * width * sizeof(mcg_bvh_node);
    const size_t b_ct = static_cast<size_t>(n) * sizeof(CollapseTask);
    auto al = [](size_t x) { return (x + 255) & ~static_cast<size_t>(255); };
    m.ensure(al(b_leaves) + 3 * al(b_idx) + 2 * al(b_tasks) + al(b_bn) + 256 + al(b_out) + 2 * al(b_ct));
    char* p = m.as<char>();
    auto take = [&](size_t b) { char* r = p; p += al(b); return r; };
    mcg_bvh_node* d_leaves = reinterpret_cast<mcg_bvh_node*>(take(b_leaves));
    int32_t* idx[2] = {reinterpret_cast<int32_t*>(take(b_idx)), reinterpret_cast<int32_t*>(take(b_idx))};
    int32_t* scratch = reinterpret_cast<int32_t*>(take(b_idx));   // partition swap ranks
    SahTask* tasks[2] = {reinterpret_cast<SahTask*>(take(b_tasks)), reinterpret_cast<SahTask*>(take(b_tasks))};
    BinNode* bn = reinterpret_cast<BinNode*>(take(b_bn));
    int32_t* counters = reinterpret_cast<int32_t*>(take(256));
    mcg_bvh_node* d_out = reinterpret_cast<mcg_bvh_node*>(take(b_out));
    CollapseTask* ct[2] = {reinterpret_cast<CollapseTask*>(take(b_ct)), reinterpret_cast<CollapseTask*>(take(b_ct))};

    std::vector<int32_t> iota(n);
    for (int i = 0; i < n; ++i) iota[i] = i;
    cuda_check(cudaMemcpyAsync(d_leaves, leaves.data(), b_leaves, cudaMemcpyHostToDevice, s), "H2D leaves");
    cuda_check(cudaMemcpyAsync(idx[0], iota.data(), b_idx, cudaMemcpyHostToDevice, s), "H2D idx");
    const SahTask root{0, 0, n, 0};
    cuda_check(cudaMemcpyAsync(tasks[0], &root, sizeof(root), cudaMemcpyHostToDevice, s), "H2D task");
    int32_t host_ctr[2] = {0, 1};   // [0] next level's tasks, [1] binary nodes allocated
    cuda_check(cudaMemcpyAsync(counters, host_ctr, 8, cudaMemcpyHostToDevice, s), "H2D counters");
    int n_tasks = 1, cur = 0;
    while (n_tasks > 0) {
        cuda_check(cudaMemsetAsync(counters, 0, 4, s), "memset counters");
        k_sah_level<<<n_tasks, kBuildBlock, 0, s>>>(d_leaves, idx[cur], idx[cur ^ 1], tasks[cur], bn,
                                                    tasks[cur ^ 1], counters, scratch);
        cuda_check(cudaGetLastError(), "k_sah_level");
        ++ctx->launches;
        cuda_check(cudaMemcpyAsync(host_ctr, counters, 8, cudaMemcpyDeviceToHost, s), "D2H counters");
        cuda_check(cudaStreamSynchronize(s), "sah level");
        n_tasks = host_ctr[0];
        cur ^= 1;
    }
    // collapse, top-down
    cuda_check(cudaMemsetAsync(d_out, 0, b_out, s), "memset");
    const CollapseTask croot{0, 0};
    cuda_check(cudaMemcpyAsync(ct[0], &croot, sizeof(croot), cudaMemcpyHostToDevice, s), "H2D task");
    int32_t cctr[2] = {0, 1};   // [0] next level's tasks, [1] output nodes allocated
    cuda_check(cudaMemcpyAsync(counters, cctr, 8, cudaMemcpyHostToDevice, s), "H2D counters");
    n_tasks = 1;
    cur = 0;
    while (n_tasks > 0) {
        cuda_check(cudaMemsetAsync(counters, 0, 4, s), "memset counters");
        k_collapse<<<grid_for(n_tasks, 128), 128, 0, s>>>(bn, d_leaves, ct[cur], n_tasks, width, d_out,
                                                          ct[cur ^ 1], counters);
        cuda_check(cudaGetLastError(), "k_collapse");
        ++ctx->launches;
        cuda_check(cudaMemcpyAsync(cctr, counters, 8, cudaMemcpyDeviceToHost, s), "D2H counters");
        cuda_check(cudaStreamSynchronize(s), "collapse level");
        n_tasks = cctr[0];
        cur ^= 1;
    }
    out.resize(static_cast<size_t>(cctr[1]) * width);
    cuda_check(cudaMemcpyAsync(out.data(), d_out, out.size() * sizeof(mcg_bvh_node), cudaMemcpyDeviceToHost, s),
               "D2H tree");
    cuda_check(cudaStreamSynchronize(s), "shadow tree");
    root_a = 0;
    root_b = -1;
    return out;
}

}  // namespace mcg

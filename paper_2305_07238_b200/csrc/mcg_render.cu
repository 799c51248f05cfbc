// Wavefront path tracer driving the material cache on the GPU: the body of
// render() (tracer.hpp:69-70, absent in the reference; restated per
// tracer.hpp:7-94 + SPEC.md:378-434 with the decisions pinned in DESIGN.md
// §render). One pass = k samples of every pixel of this shard in flight:
//
//   k_primary        camera rays, closest hit, shading record, sort key
//   per vertex b:
//     sort           (material slot | Morton code of the hit point) -> order
//     k_shade        warp-uniform bytecode VM with inline cache lookup/store
//                    (stackvm.cpp:248-368, cache.cpp:94-136), then NEE (one
//                    shadow ray per light) and the cosine bounce
//     [deterministic mode: queued stores sorted by (cell, sample, pixel,
//      ord) and applied cell by cell -- the epoch rule, DESIGN.md]
//     k_shadow_ww    any-hit of the queued shadow rays
//     k_resolve      visible light contributions, in light order
//     k_trace_closest_ww  closest hits of the continuation rays
//   k_accumulate     finished paths into the double framebuffers, samples in
//                    order (FrameBuffers, tracer.hpp:24-43)
//
// Path state moves with the sort: k_shade gathers each path's state from
// its old position and writes it at its sorted position, so every later
// kernel of the vertex reads and writes its own index (coalesced). A path's
// identity travels in `pid` (pass slot j * n_pix + pixel index); its final
// radiance lands in `fin[pid]` when it ends.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <exception>
#include <string>
#include <cstring>
#include <thread>
#include <vector>

#include "host_scene.hpp"
#include "mcg_ctx.cuh"

using namespace mcg;
using mcgd::V3;

namespace {

constexpr float kTMin = 1e-4f;
constexpr float kEps = 1e-4f;
constexpr float kInvPi = 0.318309886183790671538f;

// Render counters (device, u64): see kStat*.
enum {
    kStatLookups = 0, kStatHits, kStatWon, kStatFull, kStatLost, kStatStores, kStatInstrs,
    kStatShade, kStatShadow, kStatNodes, kStatPrims, kStatTex, kStatNodesShadow, kStatPrimsShadow,
    kStatClosestRays, kStatOccluded,
    kStatCount = 17
};

// A path's ray record (128 bytes: one line, one DRAM access when gathered):
// the ray the trace kernels read (ro.w = cone width at the origin); the
// shading point of its closest hit, written by the trace kernel that found
// it (surface, scene.cpp:211-247, and footprint gradients, raycone.cpp:50-65,
// of the cone propagated over the hit distance) -- the shade reads it instead
// of rebuilding it from the primitive; and the look-ahead probe results.
struct __align__(128) PathRay {
    float4 ro, rd;
    float4 sp0;     // hit position, propagated cone width
    float4 sp1;     // shading normal, pixel index (uint bits)
    float4 sp2;     // u, v, g1
    float4 sp3;     // g2, look-ahead flags (uint bits), -
    uint32_t ahead[8];   // look-ahead payloads (mcgd::kAhead)
};
// A path's value record (32 bytes): throughput.rgb + nodes_found (uint bits),
// radiance.rgb + path id (uint bits: pass slot j * n_pix + shard pixel index).
struct __align__(32) PathVal {
    float4 thr, L;
};

struct RenderView {
    mcgd::SceneView S;
    mcgd::CacheView C;
    int cache_on;
    int mip_offset;
    float cam[12];
    float cam_pos[3];
    int W, H;
    int max_bounces;
    unsigned long long seed;
    float diffuse_spread;
    uint32_t n_pix;           // pixels of this shard
    const uint32_t* pix;      // shard pixel indices, ascending
    uint32_t n_paths;         // n_pix * samples in this pass
    uint32_t sample0;         // sample index of pass slot 0
    uint32_t hps_base;        // hits_per_sample index of pass slot 0
    // Path state at the current layout (index = position in the last sort
    // output; the primary pass starts at pid order) and the next layout,
    // written by k_shade at the sorted position.
    // Path state in two records per layout position, so the shade's gather
    // is two random accesses (a 64-byte and a 32-byte record) instead of one
    // per field, while every other kernel reads and writes whole records:
    PathRay* pa;              // ray (origin, cone width at the origin; direction, spread), closest
                              // hit and look-ahead results -- the trace kernels' record
    PathVal* pb;              // throughput + hits, radiance + path id -- the resolve's record
    PathRay* pa2;             // the same at the next layout (written by k_shade)
    PathVal* pb2;
    float4* fin;              // by path id: final radiance.rgb, nodes_found (uint bits)
    uint32_t* keys;           // unsorted (material slot | n_programs = no hit)
    uint32_t* vals;           // unsorted layout positions
    const uint32_t* skey;     // sorted keys: hits first, in material order
    uint32_t key_shift;       // key = slot << key_shift | look-ahead hits << key_pat | Morton code
    uint32_t key_pat;         // bits below the look-ahead hit pattern (the direction/Morton part)
    uint32_t pat_mask;        // look-ahead hit bits that enter the key (0: none)
    uint32_t ahead_on;        // look-ahead probes: results in PathRay::ahead
    uint32_t ahead_fused;     // 1: the trace kernels run the look-ahead probe (no k_lookahead launch)
    uint32_t shade_perm;      // k_shade block order: block b runs sorted block (b * shade_perm) % grid (1 = in order)
    uint32_t key_dir;         // 1: a 5-bit direction class of the next bounce above the Morton code
    float box_lo[3], box_scale[3];  // scene bounds -> 8-bit grid for the Morton code
    const uint32_t* order;    // sorted layout positions
    float4* sro;              // shadow ray per (path, light): origin.xyz, t_max
    float4* srd;              // direction.xyz
    float4* scon;             // contribution.rgb, candidate flag
    uint8_t* vis;             // 1 = light visible
    uint32_t* squeue;         // compacted shadow-ray slots
    unsigned int* shadow_count;
    double* radiance;
    double* nodes_found;
    uint32_t* samples;
    unsigned long long* hps;
    unsigned long long* stats;
    mcgd::StoreQueue q;
};

__device__ __forceinline__ uint32_t dim_rect(int b, int j, int k) { return 2u + 64u * b + 2u * j + k; }
__device__ __forceinline__ uint32_t dim_bounce(int b, int k) { return 2u + 64u * b + 62u + k; }

// Sort key of a hit: material slot in the high bits (shading stays grouped by
// material), then the octant of the bounce the vertex will take, then the
// Morton code of the hit point, so rays that leave nearby points in similar
// directions -- the next closest-hit rays, and the shadow rays -- share warps
// and traverse the same BVH nodes.
__device__ __forceinline__ uint32_t spread8(uint32_t v) {
    v &= 0xffu;
    v = (v | (v << 8)) & 0x0300f00fu;
    v = (v | (v << 4)) & 0x030c30c3u;
    v = (v | (v << 2)) & 0x09249249u;
    return v;
}
__device__ __forceinline__ uint32_t sort_key(const RenderView& R, uint32_t slot, float px, float py,
                                             float pz, V3 n, uint64_t rkey, int vtx) {
    if (slot >= R.S.n_programs || R.key_shift == 0) return slot << R.key_shift;
    const float q[3] = {(px - R.box_lo[0]) * R.box_scale[0], (py - R.box_lo[1]) * R.box_scale[1],
                        (pz - R.box_lo[2]) * R.box_scale[2]};
    uint32_t c[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) c[k] = static_cast<uint32_t>(fminf(fmaxf(q[k], 0.0f), 255.0f));
    if (!R.key_dir) {
        return (slot << R.key_shift) | spread8(c[0]) | (spread8(c[1]) << 1) | (spread8(c[2]) << 2);
    }
    if (R.key_dir == 2u) {
        // Octant of the cosine bounce this vertex will take (the formula of
        // nee_bounce with fast intrinsics -- a grouping heuristic only) above
        // the Morton code: the next closest-hit rays of a warp leave nearby
        // points in similar directions.
        uint32_t oct = 0u;
        if (vtx < R.max_bounces) {
            const float r1 = mcgd::path_sample(rkey, dim_bounce(vtx, 0));
            const float r2 = mcgd::path_sample(rkey, dim_bounce(vtx, 1));
            float sphi, cphi;
            __sincosf(r1 * mcgd::kTwoPi, &sphi, &cphi);
            const float r = sqrtf(r2);
            const float lx = r * cphi, ly = r * sphi, lz = sqrtf(fmaxf(0.0f, 1.0f - r2));
            const float sign = copysignf(1.0f, n.z);
            const float a = -1.0f / (sign + n.z);
            const float bb = (n.x * n.y) * a;
            const V3 t{1.0f + ((sign * n.x) * n.x) * a, sign * bb, -sign * n.x};
            const V3 bt{bb, sign + ((n.y * n.y) * a), -n.y};
            const V3 dv = (t * lx + bt * ly) + n * lz;
            oct = (dv.x < 0.0f ? 1u : 0u) | (dv.y < 0.0f ? 2u : 0u) | (dv.z < 0.0f ? 4u : 0u);
        }
        const uint32_t mbits = R.key_pat - 3u;
        return (slot << R.key_shift) | (oct << mbits) | spread8(c[0]) | (spread8(c[1]) << 1) | (spread8(c[2]) << 2);
    }
    // Direction class of the cosine bounce this vertex will take: the
    // normal's octant and the quadrant of its azimuth sample (dims of
    // DESIGN.md §render), so rays leaving in similar directions share warps.
    const uint32_t oct = (n.x < 0.0f ? 1u : 0u) | (n.y < 0.0f ? 2u : 0u) | (n.z < 0.0f ? 4u : 0u);
    const uint32_t quad = vtx < R.max_bounces
                              ? static_cast<uint32_t>(mcgd::path_sample(rkey, dim_bounce(vtx, 0)) * 4.0f) & 3u
                              : 0u;
    const uint32_t m18 = spread8(c[0] >> 2) | (spread8(c[1] >> 2) << 1) | (spread8(c[2] >> 2) << 2);
    return (slot << R.key_shift) | (((oct << 2) | quad) << 18) | m18;
}
__device__ __forceinline__ uint32_t key_slot(const RenderView& R, uint32_t key) {
    return key >> R.key_shift;
}
__device__ __forceinline__ uint32_t no_hit_key(const RenderView& R) {
    return R.S.n_programs << R.key_shift;
}

// A primitive's geometry as the tests read it: 3 float4 (p0, e1, e2 or
// centre + radius) and the info word (sphere flag).
struct PrimG {
    float4 g0, g1, g2;
    uint32_t info;
};
__device__ __forceinline__ PrimG load_prim(const mcgd::SceneView& S, uint32_t i) {
    return PrimG{__ldg(S.prim_geom + 3 * i), __ldg(S.prim_geom + 3 * i + 1), __ldg(S.prim_geom + 3 * i + 2),
                 __ldg(S.prim_info + i)};
}
__device__ __forceinline__ bool hit_prim_g(const PrimG& P, V3 o, V3 d, float tmin, float tmax, float& t,
                                           float& b1, float& b2);

// ray_triangle (scene.cpp:58-78) / ray_sphere (scene.cpp:80-94)
__device__ __forceinline__ bool hit_prim(const mcgd::SceneView& S, uint32_t i, V3 o, V3 d,
                                         float tmin, float tmax, float& t, float& b1, float& b2) {
    const float4 g0 = __ldg(S.prim_geom + 3 * i);
    if (__ldg(S.prim_info + i) & MCG_PRIM_SPHERE) {
        const V3 oc = o - V3{g0.x, g0.y, g0.z};
        const float b = mcgd::dot(oc, d);
        const float c = mcgd::dot(oc, oc) - g0.w * g0.w;
        const float disc = b * b - c;
        if (disc < 0.0f) return false;
        const float sq = sqrtf(disc);
        float root = -b - sq;
        if (root <= tmin || root >= tmax) {
            root = -b + sq;
            if (root <= tmin || root >= tmax) return false;
        }
        t = root;
        b1 = b2 = 0.0f;
        return true;
    }
    const float4 g1 = __ldg(S.prim_geom + 3 * i + 1), g2 = __ldg(S.prim_geom + 3 * i + 2);
    const V3 p0{g0.x, g0.y, g0.z}, e1{g1.x, g1.y, g1.z}, e2{g2.x, g2.y, g2.z};
    const V3 pvec = mcgd::cross(d, e2);
    const float det = mcgd::dot(e1, pvec);
    if (fabsf(det) < 1e-12f) return false;
    const V3 tvec = o - p0;
    const float du = mcgd::dot(tvec, pvec);
#ifdef MCG_U_PRECHECK
    // (experiment, off: 653 vs 648 ms per bench render -- the early return
    // diverges inside the leaf loop) Early-out before the IEEE division, taken only where the reference's
    // u = fl(du * fl(1/det)) is certainly out of [0, 1]: the quotient
    // du/det is negative and at least 2^-60 in magnitude (so the rounded
    // product cannot underflow to -0), or it exceeds 1 + 2^-21 (two roundings
    // move it by < 2^-22 relative). Every other case takes the exact path.
    {
        const float adet = fabsf(det), adu = fabsf(du);
        const bool neg = (du < 0.0f) != (det < 0.0f) && du != 0.0f;
        if (neg && adu >= adet * 0x1p-60f) return false;
        if (!neg && adu > adet * 1.000000953674316f) return false;   // 1 + 2^-20
    }
#endif
    const float inv_det = 1.0f / det;
    const float u = du * inv_det;
    if (u < 0.0f || u > 1.0f) return false;
    const V3 qvec = mcgd::cross(tvec, e1);
    const float v = mcgd::dot(d, qvec) * inv_det;
    if (v < 0.0f || u + v > 1.0f) return false;
    const float ht = mcgd::dot(e2, qvec) * inv_det;
    if (ht <= tmin || ht >= tmax) return false;
    t = ht;
    b1 = u;
    b2 = v;
    return true;
}

// hit_prim over preloaded geometry (the same arithmetic)
__device__ __forceinline__ bool hit_prim_g(const PrimG& P, V3 o, V3 d, float tmin, float tmax, float& t,
                                           float& b1, float& b2) {
    const float4 g0 = P.g0;
    if (P.info & MCG_PRIM_SPHERE) {
        const V3 oc = o - V3{g0.x, g0.y, g0.z};
        const float b = mcgd::dot(oc, d);
        const float c = mcgd::dot(oc, oc) - g0.w * g0.w;
        const float disc = b * b - c;
        if (disc < 0.0f) return false;
        const float sq = sqrtf(disc);
        float root = -b - sq;
        if (root <= tmin || root >= tmax) {
            root = -b + sq;
            if (root <= tmin || root >= tmax) return false;
        }
        t = root;
        b1 = b2 = 0.0f;
        return true;
    }
    const float4 g1 = P.g1, g2 = P.g2;
    const V3 p0{g0.x, g0.y, g0.z}, e1{g1.x, g1.y, g1.z}, e2{g2.x, g2.y, g2.z};
    const V3 pvec = mcgd::cross(d, e2);
    const float det = mcgd::dot(e1, pvec);
    if (fabsf(det) < 1e-12f) return false;
    const V3 tvec = o - p0;
    const float du = mcgd::dot(tvec, pvec);
#ifdef MCG_U_PRECHECK
    // (experiment, off: 653 vs 648 ms per bench render -- the early return
    // diverges inside the leaf loop) Early-out before the IEEE division, taken only where the reference's
    // u = fl(du * fl(1/det)) is certainly out of [0, 1]: the quotient
    // du/det is negative and at least 2^-60 in magnitude (so the rounded
    // product cannot underflow to -0), or it exceeds 1 + 2^-21 (two roundings
    // move it by < 2^-22 relative). Every other case takes the exact path.
    {
        const float adet = fabsf(det), adu = fabsf(du);
        const bool neg = (du < 0.0f) != (det < 0.0f) && du != 0.0f;
        if (neg && adu >= adet * 0x1p-60f) return false;
        if (!neg && adu > adet * 1.000000953674316f) return false;   // 1 + 2^-20
    }
#endif
    const float inv_det = 1.0f / det;
    const float u = du * inv_det;
    if (u < 0.0f || u > 1.0f) return false;
    const V3 qvec = mcgd::cross(tvec, e1);
    const float v = mcgd::dot(d, qvec) * inv_det;
    if (v < 0.0f || u + v > 1.0f) return false;
    const float ht = mcgd::dot(e2, qvec) * inv_det;
    if (ht <= tmin || ht >= tmax) return false;
    t = ht;
    b1 = u;
    b2 = v;
    return true;
}

// Slab test of one box split into its ray-only part: E = max(tmin, entry),
// T1 = exit (fmaxf/fminf drop NaNs exactly as the reference's loop does).
// The reference's ray_aabb(ray, box, tmin, tmax) (scene.cpp:42-56) rejects
// iff fminf(tmax, T1) < E, i.e. iff T1 < E (ray-only) or tmax < E.
__device__ __forceinline__ void slab(V3 o, V3 inv, float4 lo, float4 hi, float tmin, float& E,
                                     float& T1) {
    float t0 = (lo.x - o.x) * inv.x, t1 = (hi.x - o.x) * inv.x;
    if (inv.x < 0.0f) { const float t = t0; t0 = t1; t1 = t; }
    E = fmaxf(tmin, t0);
    T1 = t1;
    t0 = (lo.y - o.y) * inv.y; t1 = (hi.y - o.y) * inv.y;
    if (inv.y < 0.0f) { const float t = t0; t0 = t1; t1 = t; }
    E = fmaxf(E, t0);
    T1 = fminf(T1, t1);
    t0 = (lo.z - o.z) * inv.z; t1 = (hi.z - o.z) * inv.z;
    if (inv.z < 0.0f) { const float t = t0; t0 = t1; t1 = t; }
    E = fmaxf(E, t0);
    T1 = fminf(T1, t1);
}

// Scene::intersect (scene.cpp:252-278) over the child-pair layout. Visit
// order and every culling decision are the reference's: its DFS pushes left
// then right and tests a node's box when the node is popped, against the
// closest hit at that moment. Here both child boxes are tested when the
// parent is expanded; the ray-only part (T1 < E) drops the child for good
// and the closest-dependent part (closest < E) is re-checked at pop time
// from the stored entry distance -- the same decision the reference makes,
// so closest-hit ties at equal t resolve identically.
__device__ bool traverse_closest(const mcgd::SceneView& S, V3 o, V3 d, float tmin, float tmax,
                                 uint32_t& prim, float& t_out, float& b1_out, float& b2_out,
                                 uint32_t& nodes_visited, uint32_t& prims_tested) {
    if (S.n_nodes == 0) return false;
    const V3 inv{1.0f / d.x, 1.0f / d.y, 1.0f / d.z};
    int32_t sa[64], sb[64];
    float se[64];
    int top = 0;
    {
        const float4 lo = __ldg(S.nodes), hi = __ldg(S.nodes + 1);
        float E, T1;
        slab(o, inv, lo, hi, tmin, E, T1);
        if (T1 < E) return false;
        // The root's own record holds its children; an internal root is
        // referenced by its index (0), a leaf root by (~first, count).
        const int32_t ra = __float_as_int(lo.w);
        sa[0] = ra >= 0 ? 0 : ra;
        sb[0] = __float_as_int(hi.w);
        se[0] = E;
        top = 1;
    }
    bool found = false;
    float closest = tmax;
    while (top > 0) {
        --top;
        const int32_t a = sa[top], b = sb[top];
        ++nodes_visited;
        if (closest < se[top]) continue;
        if (a < 0) {
            const uint32_t first = static_cast<uint32_t>(~a);
            prims_tested += static_cast<uint32_t>(b);
            for (uint32_t i = first; i < first + static_cast<uint32_t>(b); ++i) {
                float t, b1, b2;
                if (hit_prim(S, i, o, d, tmin, closest, t, b1, b2)) {
                    closest = t;
                    prim = i;
                    t_out = t;
                    b1_out = b1;
                    b2_out = b2;
                    found = true;
                }
            }
        } else {
            const float4* p = S.pairs + 4 * a;
            const float4 llo = __ldg(p), lhi = __ldg(p + 1), rlo = __ldg(p + 2), rhi = __ldg(p + 3);
            float EL, T1L, ER, T1R;
            slab(o, inv, llo, lhi, tmin, EL, T1L);
            slab(o, inv, rlo, rhi, tmin, ER, T1R);
            if (!(T1L < EL)) {
                sa[top] = __float_as_int(llo.w);
                sb[top] = __float_as_int(lhi.w);
                se[top] = EL;
                ++top;
            }
            if (!(T1R < ER)) {
                sa[top] = __float_as_int(rlo.w);
                sb[top] = __float_as_int(rhi.w);
                se[top] = ER;
                ++top;
            }
        }
    }
    return found;
}

// Scene::occluded (scene.cpp:280-298): a boolean whose value does not depend
// on visit order (tmax is fixed), so children are visited near-first and the
// far one is stacked; the first hit ends the query.
__device__ bool traverse_any(const mcgd::SceneView& S, V3 o, V3 d, float tmin, float tmax,
                             uint32_t& nodes_visited, uint32_t& prims_tested) {
    if (S.n_nodes == 0) return false;
    const V3 inv{1.0f / d.x, 1.0f / d.y, 1.0f / d.z};
    int32_t sa[64], sb[64];
    int top = 0;
    int32_t a, b;
    {
        const float4 lo = __ldg(S.nodes), hi = __ldg(S.nodes + 1);
        float E, T1;
        slab(o, inv, lo, hi, tmin, E, T1);
        if (fminf(tmax, T1) < E) return false;
        a = __float_as_int(lo.w);
        a = a >= 0 ? 0 : a;
        b = __float_as_int(hi.w);
    }
    for (;;) {
        ++nodes_visited;
        if (a < 0) {
            const uint32_t first = static_cast<uint32_t>(~a);
            prims_tested += static_cast<uint32_t>(b);
            for (uint32_t i = first; i < first + static_cast<uint32_t>(b); ++i) {
                float t, b1, b2;
                if (hit_prim(S, i, o, d, tmin, tmax, t, b1, b2)) return true;
            }
            if (top == 0) return false;
            --top;
            a = sa[top];
            b = sb[top];
            continue;
        }
        const float4* p = S.pairs + 4 * a;
        const float4 llo = __ldg(p), lhi = __ldg(p + 1), rlo = __ldg(p + 2), rhi = __ldg(p + 3);
        float EL, T1L, ER, T1R;
        slab(o, inv, llo, lhi, tmin, EL, T1L);
        slab(o, inv, rlo, rhi, tmin, ER, T1R);
        const bool okL = !(fminf(tmax, T1L) < EL), okR = !(fminf(tmax, T1R) < ER);
        if (okL && okR) {
            const bool left_first = EL <= ER;
            sa[top] = __float_as_int(left_first ? rlo.w : llo.w);
            sb[top] = __float_as_int(left_first ? rhi.w : lhi.w);
            ++top;
            a = __float_as_int(left_first ? llo.w : rlo.w);
            b = __float_as_int(left_first ? lhi.w : rhi.w);
        } else if (okL || okR) {
            a = __float_as_int(okL ? llo.w : rlo.w);
            b = __float_as_int(okL ? lhi.w : rhi.w);
        } else {
            if (top == 0) return false;
            --top;
            a = sa[top];
            b = sb[top];
        }
    }
}

struct Surface {
    V3 p, n;
    float u, v;
    V3 e1, e2;
    float2 d1, d2;
    uint32_t slot;
};

// HitRecord construction (scene.cpp:211-247).
__device__ Surface surface(const mcgd::SceneView& S, V3 o, V3 d, uint32_t prim, float t, float b1,
                           float b2) {
    Surface s;
    const uint32_t info = __ldg(S.prim_info + prim);
    s.slot = info & ~MCG_PRIM_SPHERE;
    s.p = o + d * t;
    const float4 g0 = __ldg(S.prim_geom + 3 * prim);
    if (!(info & MCG_PRIM_SPHERE)) {
        const float4 g1 = __ldg(S.prim_geom + 3 * prim + 1), g2 = __ldg(S.prim_geom + 3 * prim + 2);
        s.e1 = V3{g1.x, g1.y, g1.z};
        s.e2 = V3{g2.x, g2.y, g2.z};
        V3 n = mcgd::normalize(mcgd::cross(s.e1, s.e2));
        if (mcgd::dot(n, d) > 0.0f) n = V3{-n.x, -n.y, -n.z};
        s.n = n;
        const float2 uv0 = __ldg(S.prim_uv + 3 * prim), uv1 = __ldg(S.prim_uv + 3 * prim + 1),
                     uv2 = __ldg(S.prim_uv + 3 * prim + 2);
        const float w0 = 1.0f - b1 - b2;
        s.u = uv0.x * w0 + uv1.x * b1 + uv2.x * b2;
        s.v = uv0.y * w0 + uv1.y * b1 + uv2.y * b2;
        s.d1 = make_float2(uv1.x - uv0.x, uv1.y - uv0.y);
        s.d2 = make_float2(uv2.x - uv0.x, uv2.y - uv0.y);
        return s;
    }
    // Sphere (scene.cpp:227-246). atan2f/acosf: the deterministic routines
    // the oracle uses (device_math.cuh), within 1 ulp of glibc's.
    const float kPi = 3.14159265358979323846f;
    const V3 m = mcgd::normalize(s.p - V3{g0.x, g0.y, g0.z});
    V3 n = m;
    if (mcgd::dot(n, d) > 0.0f) n = V3{-n.x, -n.y, -n.z};
    s.n = n;
    s.u = 0.5f + mcgd::det_atan2f(m.z, m.x) / (2.0f * kPi);
    s.v = mcgd::det_acosf(fminf(fmaxf(m.y, -1.0f), 1.0f)) / kPi;
    const float sin_t = sqrtf(fmaxf(0.0f, 1.0f - m.y * m.y));
    const float r = g0.w;
    if (sin_t > 1e-6f) {
        s.e1 = V3{-m.z, 0.0f, m.x} * (2.0f * kPi * r);
        const float cphi = m.x / sin_t, sphi = m.z / sin_t;
        s.e2 = V3{m.y * cphi, -sin_t, m.y * sphi} * (kPi * r);
    } else {
        s.e1 = V3{1.0f, 0.0f, 0.0f} * (2.0f * kPi * r);
        s.e2 = V3{0.0f, 0.0f, 1.0f} * (kPi * r);
    }
    s.d1 = make_float2(1.0f, 0.0f);
    s.d2 = make_float2(0.0f, 1.0f);
    return s;
}

// Camera ray of path i (camera).
__device__ __forceinline__ void camera_ray(const RenderView& R, uint32_t pixel, uint64_t rkey,
                                           V3& o, V3& d) {
    const int x = static_cast<int>(pixel % static_cast<uint32_t>(R.W));
    const int y = static_cast<int>(pixel / static_cast<uint32_t>(R.W));
    const float jx = mcgd::path_sample(rkey, 0), jy = mcgd::path_sample(rkey, 1);
    const float sx = ((static_cast<float>(x) + jx) / static_cast<float>(R.W)) * 2.0f - 1.0f;
    const float sy = 1.0f - ((static_cast<float>(y) + jy) / static_cast<float>(R.H)) * 2.0f;
    const float a = (sx * R.cam[9]) * R.cam[10];
    const float bq = sy * R.cam[9];
    const V3 fwd{R.cam[0], R.cam[1], R.cam[2]}, right{R.cam[3], R.cam[4], R.cam[5]},
        up{R.cam[6], R.cam[7], R.cam[8]};
    o = V3{R.cam_pos[0], R.cam_pos[1], R.cam_pos[2]};
    d = mcgd::normalize((fwd + right * a) + up * bq);
}

// The look-ahead probe of the live hit at layout position q with shading
// point `in` (k_lookahead below): its material's first kAhead cache points,
// results to R.ahead[q]; returns the sort key with the hit bits added.
// kMax: the kernel's bound on the cache points probed (3 when no material of
// the scene has more: the loop unrolls, as the one-bracket scenes want)
template <uint32_t kMax>
__device__ __forceinline__ uint32_t look_ahead(const RenderView& R, uint32_t q, uint32_t key,
                                               const mcgd::ShadeIn& in) {
    uint32_t flags = 0u;
    const uint32_t slot = key_slot(R, key);
    const mcg_program prog = R.S.programs[slot];
    const uint32_t ncp = min(prog.cache_point_count, kMax);
    PathRay& rec = R.pa[q];
    uint32_t kbits = 0u;   // hit bits of the table's first two entries (the sort key's)
    const uint32_t mip = mcgd::mip_level(in.g1x, in.g1y, in.g2x, in.g2y, R.mip_offset);
    const uint32_t tx = mcgd::texel_index(in.u, mip), ty = mcgd::texel_index(in.v, mip);
    auto probe = [&](uint32_t c) {
        const uint2 cp = __ldg(R.S.ahead_cp + slot * mcgd::kAhead + c);
        mcgd::Desc desc{prog.material_id, cp.x, 0u, 0u, 0u};
        if (cp.y & MCG_F_USES_UV) {
            desc.mip = mip;
            desc.tx = tx;
            desc.ty = ty;
        }
        uint64_t h;
        uint32_t check;
        mcgd::hash_desc(desc, h, check);
        // the whole cell in one round trip (head block + first tail pair): the
        // epilogue has bandwidth to spare, and a filling table makes most
        // scans run past the first pair
        const mcgd::Probe pr = mcgd::probe_cell_t<5>(R.C, mcgd::fast_mod(h, R.C.n_cells, R.C.magic), check);
        const uint32_t bi = (cp.y >> 16) & 0xffu;   // the bracket: flag bits and payloads are by bracket
        if (pr.hit) {
            flags |= 1u << bi;
            rec.ahead[bi] = pr.payload;
            if (c < 2u) kbits |= 1u << c;
        } else if (pr.where < 0) {
            flags |= 1u << (mcgd::kAheadFull + bi);
        }
    };
    // unrolled for the short bound only (an unrolled eight-step loop made the
    // many-cache-point kernels 15% slower; a rolled three-step loop the
    // one-bracket bench 1.3% slower)
    if constexpr (kMax <= 3u) {
#pragma unroll
        for (uint32_t c = 0; c < kMax; ++c) {
            if (c >= ncp) break;
            probe(c);
        }
    } else {
#pragma unroll 1
        for (uint32_t c = 0; c < ncp; ++c) probe(c);
    }
    rec.sp3.z = __uint_as_float(flags);
    return key | ((kbits & R.pat_mask) << R.key_pat);
}

// Closest hit of the path at layout position q (path id pid): the hit
// record (primitive, t, barycentrics: 16 bytes) at q, the propagated cone
// width into ro.w, and the sort key; on a miss the path ends: radiance +
// throughput * env goes to fin[pid] and the key is "no hit". k_shade
// rebuilds the shading record (position, normal, uv, footprint gradients)
// from the hit record with the same arithmetic (shade_input), so one 16-byte
// gather replaces three.
template <uint32_t kMax>
__device__ __forceinline__ uint32_t hit_record(const RenderView& R, uint32_t q, uint32_t pid, float4& ro,
                                               const float4& rd, const float4& thr, const float4& L,
                                               bool found, uint32_t prim, float t, float b1, float b2,
                                               int vtx) {
    const V3 o{ro.x, ro.y, ro.z}, d{rd.x, rd.y, rd.z};
    if (!found) {
        R.fin[pid] = make_float4(L.x + thr.x * R.S.env[0], L.y + thr.y * R.S.env[1],
                                 L.z + thr.z * R.S.env[2], thr.w);
        return no_hit_key(R);
    }
    const Surface s = surface(R.S, o, d, prim, t, b1, b2);
    ro.w = ro.w + t * rd.w;  // propagate (raycone.cpp:15-18)
    const uint32_t slot_j = pid / R.n_pix;
    const uint32_t pixel = R.pix[pid - slot_j * R.n_pix];
    const uint64_t rkey = mcgd::path_key(R.seed, pixel, R.sample0 + slot_j);
    const uint32_t key = sort_key(R, s.slot, s.p.x, s.p.y, s.p.z, s.n, rkey, vtx);
    // the shading point (ShadingPoint, geom.hpp:49-56) for the shade
    float2 g1, g2;
    mcgd::footprint(ro.w, d, s.n, s.e1, s.e2, s.d1, s.d2, g1, g2);
    PathRay& rec = R.pa[q];
    rec.sp0 = make_float4(s.p.x, s.p.y, s.p.z, ro.w);
    rec.sp1 = make_float4(s.n.x, s.n.y, s.n.z, __uint_as_float(pixel));
    rec.sp2 = make_float4(s.u, s.v, g1.x, g1.y);
    rec.sp3 = make_float4(g2.x, g2.y, __uint_as_float(0u), 0.0f);
    if (!R.ahead_fused || s.slot >= R.S.n_programs) return key;
    // the look-ahead probes right here (a separate kernel for the cache
    // points past the first two, after the trace, measured slower: monster
    // analogue 1363 vs 1285 ms per render)
    const mcgd::ShadeIn in{s.p.x, s.p.y, s.p.z, s.n.x, s.n.y, s.n.z, d.x, d.y, d.z,
                           s.u, s.v, g1.x, g1.y, g2.x, g2.y};
    return look_ahead<kMax>(R, q, key, in);
}

// The shading point the trace kernel stored in a path's ray record.
__device__ __forceinline__ mcgd::ShadeIn shade_input(const float4& rd, const float4& sp0, const float4& sp1,
                                                     const float4& sp2, const float4& sp3) {
    return mcgd::ShadeIn{sp0.x, sp0.y, sp0.z, sp1.x, sp1.y, sp1.z, rd.x, rd.y, rd.z,
                         sp2.x, sp2.y, sp2.z, sp2.w, sp3.x, sp3.y};
}

// Next-event estimation and the cosine bounce of vertex b of path pid, whose
// state goes to sorted position i: one shadow-ray candidate per light -- its
// contribution computed now, applied in light order by k_resolve once
// visibility is known -- and the continuation ray.
__device__ __forceinline__ void nee_bounce(const RenderView& R, uint32_t i, uint32_t pid, uint32_t pixel, int b,
                                           V3 pos, V3 n, float3 bc, float4 thr, float width, float spread) {
    const uint32_t slot_j = pid / R.n_pix;
    const uint64_t rkey = mcgd::path_key(R.seed, pixel, R.sample0 + slot_j);
    const V3 alb{fminf(fmaxf(bc.x, 0.0f), 1.0f), fminf(fmaxf(bc.y, 0.0f), 1.0f),
                 fminf(fmaxf(bc.z, 0.0f), 1.0f)};
    const V3 f = alb * kInvPi;
    const V3 tf{thr.x * f.x, thr.y * f.y, thr.z * f.z};
    const V3 o = pos + n * kEps;
    const uint32_t nl = R.S.n_plights + R.S.n_rlights;
    const unsigned lane = threadIdx.x & 31u;
    for (uint32_t j = 0; j < nl; ++j) {
        const uint32_t s = i * nl + j;
        bool cand = false;
        V3 wi{0.0f, 0.0f, 0.0f};
        float dist = 0.0f, w = 0.0f;
        const float* emit;
        if (j < R.S.n_plights) {
            const mcg_point_light& l = R.S.plights[j];
            const V3 toL = V3{l.position[0], l.position[1], l.position[2]} - o;
            const float d2 = mcgd::dot(toL, toL);
            dist = sqrtf(d2);
            wi = toL * (1.0f / dist);
            const float cs = mcgd::dot(n, wi);
            cand = cs > 0.0f;
            w = cs / d2;
            emit = l.intensity;
        } else {
            const uint32_t jr = j - R.S.n_plights;
            const mcg_rect_light& l = R.S.rlights[jr];
            const float u = mcgd::path_sample(rkey, dim_rect(b, static_cast<int>(jr), 0));
            const float vv = mcgd::path_sample(rkey, dim_rect(b, static_cast<int>(jr), 1));
            const V3 eu{l.edge_u[0], l.edge_u[1], l.edge_u[2]};
            const V3 ev{l.edge_v[0], l.edge_v[1], l.edge_v[2]};
            const V3 pl = (V3{l.corner[0], l.corner[1], l.corner[2]} + eu * u) + ev * vv;
            const V3 nlv = mcgd::cross(eu, ev);
            const float area = mcgd::length(nlv);
            const V3 toL = pl - o;
            const float d2 = mcgd::dot(toL, toL);
            dist = sqrtf(d2);
            wi = toL * (1.0f / dist);
            const float cs = mcgd::dot(n, wi);
            const float cl = fabsf(mcgd::dot(nlv, wi)) / area;
            cand = cs > 0.0f && cl > 0.0f;
            w = ((cs * cl) * area) / d2;
            emit = l.radiance;
        }
        if (cand) {
            R.sro[s] = make_float4(o.x, o.y, o.z, dist);
            R.srd[s] = make_float4(wi.x, wi.y, wi.z, 0.0f);
            R.scon[s] = make_float4(tf.x * (emit[0] * w), tf.y * (emit[1] * w), tf.z * (emit[2] * w), 1.0f);
        } else {
            R.scon[s] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        }
        // Append to the shadow-ray queue: one atomic per warp.
        const unsigned act = __activemask();
        const unsigned m = __ballot_sync(act, cand);
        if (m) {
            const int ldr = __ffs(m) - 1;
            unsigned basepos = 0;
            if (static_cast<int>(lane) == ldr) basepos = atomicAdd(R.shadow_count, static_cast<unsigned>(__popc(m)));
            basepos = __shfl_sync(act, basepos, ldr);
            MCG_CHECK(!cand || basepos + __popc(m & ((1u << lane) - 1u)) < R.n_paths * nl);
            if (cand) R.squeue[basepos + __popc(m & ((1u << lane) - 1u))] = s;
        }
    }
    if (b < R.max_bounces) {
        // Cosine-weighted bounce in Duff et al.'s branchless frame.
        const float r1 = mcgd::path_sample(rkey, dim_bounce(b, 0));
        const float r2 = mcgd::path_sample(rkey, dim_bounce(b, 1));
        float sphi, cphi;
        mcgd::det_sincosf(r1 * mcgd::kTwoPi, sphi, cphi);
        const float r = sqrtf(r2);
        const float lx = r * cphi, ly = r * sphi;
        const float lz = sqrtf(fmaxf(0.0f, 1.0f - r2));
        const float sign = copysignf(1.0f, n.z);
        const float a = -1.0f / (sign + n.z);
        const float bb = (n.x * n.y) * a;
        const V3 t{1.0f + ((sign * n.x) * n.x) * a, sign * bb, -sign * n.x};
        const V3 bt{bb, sign + ((n.y * n.y) * a), -n.y};
        const V3 nd = mcgd::normalize((t * lx + bt * ly) + n * lz);
        thr.x = thr.x * alb.x;
        thr.y = thr.y * alb.y;
        thr.z = thr.z * alb.z;
        R.pa2[i].ro = make_float4(o.x, o.y, o.z, width);
        R.pa2[i].rd = make_float4(nd.x, nd.y, nd.z, spread + R.diffuse_spread);  // widen
    }
    R.pb2[i].thr = thr;
}

// ---------------------------------------------------------------------------
// Warp-synchronous "while-while" traversal. Each lane walks its own ray in
// exactly the order traverse_closest / traverse_any use; a lane that pops a
// leaf parks on it until every lane of the warp holds a leaf or is done,
// then all parked lanes test their triangles together. Leaf tests (the
// expensive part) therefore run with most lanes active instead of a couple,
// and no lane ever runs ahead of its own reference order. Every lane of the
// warp must call these (inactive lanes pass active = false).
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool closest_ww(const mcgd::SceneView& S, bool active, V3 o, V3 d,
                                           float tmin, float tmax, uint32_t& prim, float& t_out,
                                           float& b1_out, float& b2_out, uint32_t& nodes_visited,
                                           uint32_t& prims_tested) {
    const V3 inv{1.0f / d.x, 1.0f / d.y, 1.0f / d.z};
    int32_t sa[64], sb[64];
    float se[64];
    int top = 0;
    if (active && S.n_nodes) {
        const float4 lo = __ldg(S.nodes), hi = __ldg(S.nodes + 1);
        float E, T1;
        slab(o, inv, lo, hi, tmin, E, T1);
        if (!(T1 < E)) {
            const int32_t ra = __float_as_int(lo.w);
            sa[0] = ra >= 0 ? 0 : ra;
            sb[0] = __float_as_int(hi.w);
            se[0] = E;
            top = 1;
        }
    }
    bool found = false;
    float closest = tmax;
    int32_t la = 0, lb = 0;
    bool leaf = false;
    bool done = top == 0;
    while (__any_sync(mcgd::kFull, !done)) {
        // Phase 1: pop and expand until this lane holds a leaf (or is done).
        for (;;) {
            if (!done && !leaf) {
                if (top == 0) {
                    done = true;
                } else {
                    --top;
                    const int32_t a = sa[top], b = sb[top];
                    ++nodes_visited;
                    if (!(closest < se[top])) {
                        if (a < 0) {
                            leaf = true;
                            la = a;
                            lb = b;
                        } else {
                            const float4* p = S.pairs + 4 * a;
                            const float4 llo = __ldg(p), lhi = __ldg(p + 1), rlo = __ldg(p + 2), rhi = __ldg(p + 3);
                            float EL, T1L, ER, T1R;
                            slab(o, inv, llo, lhi, tmin, EL, T1L);
                            slab(o, inv, rlo, rhi, tmin, ER, T1R);
                            if (!(T1L < EL)) {
                                sa[top] = __float_as_int(llo.w);
                                sb[top] = __float_as_int(lhi.w);
                                se[top] = EL;
                                ++top;
                            }
                            if (!(T1R < ER)) {
                                sa[top] = __float_as_int(rlo.w);
                                sb[top] = __float_as_int(rhi.w);
                                se[top] = ER;
                                ++top;
                            }
                        }
                    }
                }
            }
            if (__all_sync(mcgd::kFull, done || leaf)) break;
        }
        // Phase 2: every parked lane tests its leaf (the reference's order).
        if (leaf) {
            const uint32_t first = static_cast<uint32_t>(~la);
            prims_tested += static_cast<uint32_t>(lb);
            for (uint32_t i = first; i < first + static_cast<uint32_t>(lb); ++i) {
                float t, b1, b2;
                if (hit_prim(S, i, o, d, tmin, closest, t, b1, b2)) {
                    closest = t;
                    prim = i;
                    t_out = t;
                    b1_out = b1;
                    b2_out = b2;
                    found = true;
                }
            }
            leaf = false;
            done = top == 0;
        }
    }
    return found;
}

__device__ __forceinline__ bool any_ww(const mcgd::SceneView& S, bool active, V3 o, V3 d, float tmin,
                                       float tmax, uint32_t& nodes_visited, uint32_t& prims_tested) {
    const V3 inv{1.0f / d.x, 1.0f / d.y, 1.0f / d.z};
    int32_t sa[64], sb[64];
    int top = 0;
    if (active && S.n_nodes) {
        const float4 lo = __ldg(S.nodes), hi = __ldg(S.nodes + 1);
        float E, T1;
        slab(o, inv, lo, hi, tmin, E, T1);
        if (!(fminf(tmax, T1) < E)) {
            const int32_t ra = __float_as_int(lo.w);
            sa[0] = ra >= 0 ? 0 : ra;
            sb[0] = __float_as_int(hi.w);
            top = 1;
        }
    }
    bool hit = false;
    int32_t la = 0, lb = 0;
    bool leaf = false;
    bool done = top == 0;
    while (__any_sync(mcgd::kFull, !done)) {
        for (;;) {
            if (!done && !leaf) {
                if (top == 0) {
                    done = true;
                } else {
                    --top;
                    const int32_t a = sa[top], b = sb[top];
                    ++nodes_visited;
                    if (a < 0) {
                        leaf = true;
                        la = a;
                        lb = b;
                    } else {
                        const float4* p = S.pairs + 4 * a;
                        const float4 llo = __ldg(p), lhi = __ldg(p + 1), rlo = __ldg(p + 2), rhi = __ldg(p + 3);
                        float EL, T1L, ER, T1R;
                        slab(o, inv, llo, lhi, tmin, EL, T1L);
                        slab(o, inv, rlo, rhi, tmin, ER, T1R);
                        const bool okL = !(fminf(tmax, T1L) < EL), okR = !(fminf(tmax, T1R) < ER);
                        // far child first so the near one is popped next
                        const bool lf = EL <= ER;
                        if (lf ? okR : okL) {
                            sa[top] = __float_as_int(lf ? rlo.w : llo.w);
                            sb[top] = __float_as_int(lf ? rhi.w : lhi.w);
                            ++top;
                        }
                        if (lf ? okL : okR) {
                            sa[top] = __float_as_int(lf ? llo.w : rlo.w);
                            sb[top] = __float_as_int(lf ? lhi.w : rhi.w);
                            ++top;
                        }
                    }
                }
            }
            if (__all_sync(mcgd::kFull, done || leaf)) break;
        }
        if (leaf) {
            const uint32_t first = static_cast<uint32_t>(~la);
            prims_tested += static_cast<uint32_t>(lb);
            for (uint32_t i = first; i < first + static_cast<uint32_t>(lb); ++i) {
                float t, b1, b2;
                if (hit_prim(S, i, o, d, tmin, tmax, t, b1, b2)) {
                    hit = true;
                    break;
                }
            }
            leaf = false;
            done = hit || top == 0;
        }
    }
    return hit;
}

// ---------------------------------------------------------------------------
// 4-wide variants over the collapsed tree (SceneView::quads). A popped
// 4-wide node pushes its (up to four) entries -- the reference's
// grandchildren -- in left-to-right order, so the LIFO visit order is the
// reference's; each entry's box test is split into its ray-only part (at
// push) and the closest-dependent part (at pop), as in closest_ww.
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool closest_ww4(const mcgd::SceneView& S, bool active, V3 o, V3 d,
                                            float tmin, float tmax, uint32_t& prim, float& t_out,
                                            float& b1_out, float& b2_out, uint32_t& nodes_visited,
                                            uint32_t& prims_tested) {
    const V3 inv{1.0f / d.x, 1.0f / d.y, 1.0f / d.z};
    int32_t sa[64], sb[64];
    float se[64];
    int top = 0;
    if (active && S.n_nodes) {
        const float4 lo = __ldg(S.nodes), hi = __ldg(S.nodes + 1);
        float E, T1;
        slab(o, inv, lo, hi, tmin, E, T1);
        if (!(T1 < E)) {
            sa[0] = S.root_a;
            sb[0] = S.root_b;
            se[0] = E;
            top = 1;
        }
    }
    bool found = false;
    float closest = tmax;
    int32_t la = 0, lb = 0;
    bool leaf = false;
    bool done = top == 0;
    while (__any_sync(mcgd::kFull, !done)) {
        for (;;) {
            if (!done && !leaf) {
                if (top == 0) {
                    done = true;
                } else {
                    --top;
                    const int32_t a = sa[top], b = sb[top];
                    ++nodes_visited;
                    if (!(closest < se[top])) {
                        if (b > 0) {
                            leaf = true;
                            la = a;
                            lb = b;
                        } else {
                            const float4* p = S.quads + 2 * mcgd::kClosestWidth * a;
#pragma unroll
                            for (int k = 0; k < mcgd::kClosestWidth; ++k) {
                                const float4 lo = __ldg(p + 2 * k), hi = __ldg(p + 2 * k + 1);
                                const int32_t eb = __float_as_int(hi.w);
                                if (eb == 0) continue;  // empty entry
                                float E, T1;
                                slab(o, inv, lo, hi, tmin, E, T1);
                                if (!(T1 < E)) {
                                    sa[top] = __float_as_int(lo.w);
                                    sb[top] = eb;
                                    se[top] = E;
                                    ++top;
                                }
                            }
                        }
                    }
                }
            }
            if (__all_sync(mcgd::kFull, done || leaf)) break;
        }
        if (leaf) {
            const uint32_t first = static_cast<uint32_t>(~la);
            prims_tested += static_cast<uint32_t>(lb);
            for (uint32_t i = first; i < first + static_cast<uint32_t>(lb); ++i) {
                float t, b1, b2;
                if (hit_prim(S, i, o, d, tmin, closest, t, b1, b2)) {
                    closest = t;
                    prim = i;
                    t_out = t;
                    b1_out = b1;
                    b2_out = b2;
                    found = true;
                }
            }
            leaf = false;
            done = top == 0;
        }
    }
    return found;
}

__device__ __forceinline__ bool any_ww4(const mcgd::SceneView& S, bool active, V3 o, V3 d, float tmin,
                                        float tmax, uint32_t& nodes_visited, uint32_t& prims_tested) {
    const V3 inv{1.0f / d.x, 1.0f / d.y, 1.0f / d.z};
    int32_t sa[64], sb[64];
    int top = 0;
    if (active && S.n_nodes) {
        const float4 lo = __ldg(S.nodes), hi = __ldg(S.nodes + 1);
        float E, T1;
        slab(o, inv, lo, hi, tmin, E, T1);
        if (!(fminf(tmax, T1) < E)) {
            sa[0] = S.root_a;
            sb[0] = S.root_b;
            top = 1;
        }
    }
    bool hit = false;
    int32_t la = 0, lb = 0;
    bool leaf = false;
    bool done = top == 0;
    while (__any_sync(mcgd::kFull, !done)) {
        for (;;) {
            if (!done && !leaf) {
                if (top == 0) {
                    done = true;
                } else {
                    --top;
                    const int32_t a = sa[top], b = sb[top];
                    ++nodes_visited;
                    if (b > 0) {
                        leaf = true;
                        la = a;
                        lb = b;
                    } else {
                        // surviving entries in entry order (any order is exact for any-hit)
                        const float4* p = S.quads + 2 * mcgd::kClosestWidth * a;
#pragma unroll
                        for (int k = 0; k < mcgd::kClosestWidth; ++k) {
                            const float4 lo = __ldg(p + 2 * k), hi = __ldg(p + 2 * k + 1);
                            const int32_t eb = __float_as_int(hi.w);
                            if (eb == 0) break;
                            float E, T1;
                            slab(o, inv, lo, hi, tmin, E, T1);
                            if (!(fminf(tmax, T1) < E)) {
                                sa[top] = __float_as_int(lo.w);
                                sb[top] = eb;
                                ++top;
                            }
                        }
                    }
                }
            }
            if (__all_sync(mcgd::kFull, done || leaf)) break;
        }
        if (leaf) {
            const uint32_t first = static_cast<uint32_t>(~la);
            prims_tested += static_cast<uint32_t>(lb);
            for (uint32_t i = first; i < first + static_cast<uint32_t>(lb); ++i) {
                float t, b1, b2;
                if (hit_prim(S, i, o, d, tmin, tmax, t, b1, b2)) {
                    hit = true;
                    break;
                }
            }
            leaf = false;
            done = hit || top == 0;
        }
    }
    return hit;
}


// ---------------------------------------------------------------------------
// Four boxes at a time with packed f32x2 arithmetic (Blackwell FADD2/FMUL2,
// round-to-nearest per element: bit for bit the scalar operations) over the
// transposed 4-wide nodes (SceneView::quads_soa / squads_soa). The near and
// far plane of each axis are picked by address from the ray's direction
// signs -- the reference's swap of (lo - o) * inv and (hi - o) * inv when
// inv < 0 -- so a node costs 12 packed sub/mul pairs instead of 48 scalar
// operations and 24 selects.
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long f2sub(unsigned long long a, unsigned long long b) {
    unsigned long long r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ unsigned long long f2mul(unsigned long long a, unsigned long long b) {
    unsigned long long r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ unsigned long long f2splat(float f) {
    const unsigned long long u = __float_as_uint(f);
    return (u << 32) | u;
}
__device__ __forceinline__ float f2lo(unsigned long long v) { return __uint_as_float(static_cast<uint32_t>(v)); }
__device__ __forceinline__ float f2hi(unsigned long long v) { return __uint_as_float(static_cast<uint32_t>(v >> 32)); }

struct RayQ {
    unsigned long long ox, oy, oz;  // origin, splatted
    unsigned long long ix, iy, iz;  // 1 / direction, splatted
    int nx, ny, nz;                 // rows of the near planes (lo: 0-2, hi: 3-5)
};
__device__ __forceinline__ RayQ make_rayq(V3 o, V3 inv) {
    RayQ r;
    r.ox = f2splat(o.x);
    r.oy = f2splat(o.y);
    r.oz = f2splat(o.z);
    r.ix = f2splat(inv.x);
    r.iy = f2splat(inv.y);
    r.iz = f2splat(inv.z);
    r.nx = inv.x < 0.0f ? 3 : 0;
    r.ny = inv.y < 0.0f ? 4 : 1;
    r.nz = inv.z < 0.0f ? 5 : 2;
    return r;
}
// Entry distance E = max(tmin, near planes) and exit T1 = min(far planes)
// of the four boxes of a transposed node (the slab() split, per box), axis
// by axis so few packed values are live at once.
__device__ __forceinline__ void box4_axis(const ulonglong2* q, int near_row, unsigned long long o2,
                                          unsigned long long i2, float N[4], float F[4]) {
    const ulonglong2 n = __ldg(q + near_row), f = __ldg(q + (near_row >= 3 ? near_row - 3 : near_row + 3));
    const unsigned long long n01 = f2mul(f2sub(n.x, o2), i2), n23 = f2mul(f2sub(n.y, o2), i2);
    const unsigned long long f01 = f2mul(f2sub(f.x, o2), i2), f23 = f2mul(f2sub(f.y, o2), i2);
    N[0] = f2lo(n01);
    N[1] = f2hi(n01);
    N[2] = f2lo(n23);
    N[3] = f2hi(n23);
    F[0] = f2lo(f01);
    F[1] = f2hi(f01);
    F[2] = f2lo(f23);
    F[3] = f2hi(f23);
}
__device__ __forceinline__ void box4(const float4* node, const RayQ& r, float tmin, float E[4], float T1[4]) {
    const ulonglong2* q = reinterpret_cast<const ulonglong2*>(node);
    float N[4], F[4];
    box4_axis(q, r.nx, r.ox, r.ix, N, F);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        E[k] = fmaxf(tmin, N[k]);
        T1[k] = F[k];
    }
    box4_axis(q, r.ny, r.oy, r.iy, N, F);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        E[k] = fmaxf(E[k], N[k]);
        T1[k] = fminf(T1[k], F[k]);
    }
    box4_axis(q, r.nz, r.oz, r.iz, N, F);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        E[k] = fmaxf(E[k], N[k]);
        T1[k] = fminf(T1[k], F[k]);
    }
}

// ---------------------------------------------------------------------------
// 4-wide traversal with speculative expansion and one-word stack entries.
// An entry is (code, E): code >= 0 a 4-wide node, code < 0 a leaf
// ~(first << 3 | count) (reference leaves hold <= 4 primitives,
// scene.cpp:168). The entry to be popped next stays in registers (the last
// child pushed), so most pops never touch the local-memory stack.
//
// Speculation: a lane that already holds a leaf keeps popping while other
// lanes of its warp are still searching for theirs -- internal entries are
// expanded, the next leaf is left in place until the leaf tests ran. This
// is exact. An internal entry passes its cull test (closest < E) against a
// closest that is at least the reference's at that point, so it may be
// expanded where the reference would have culled it; but each child box lies
// inside its parent's, so every child's entry distance is >= the parent's
// (slab arithmetic is monotone under IEEE rounding) and every
// one of them is then culled when popped, against a closest that is by then
// at most the reference's. Leaves are only tested after a cull test against
// the up-to-date closest, in the reference's LIFO order.
// ---------------------------------------------------------------------------
// Leaves a lane may hold while it speculates (2: the second waits for the
// first's tests and then re-does its cull test; 743 vs 752 ms per render).
#ifndef MCG_CLOSEST_LEAVES
#define MCG_CLOSEST_LEAVES 2
#endif
__device__ __forceinline__ int32_t entry_code(int32_t a, int32_t b) {
    // quads entry (a, b): b > 0 leaf (a = ~first, b = count), b < 0 node a
    return b > 0 ? static_cast<int32_t>(~((static_cast<uint32_t>(~a) << 3) | static_cast<uint32_t>(b))) : a;
}

// A leaf's primitives in the reference's order (closest hit, strict <).
// MCG_TRI_PREFETCH=1 (experiment, off): the next primitive's geometry is
// loaded before the current one is tested (same arithmetic, same order);
// measured 652.5 vs 646.8 ms per bench render -- the extra live registers
// spill at the kernel's 64-register budget.
#ifndef MCG_TRI_PREFETCH
#define MCG_TRI_PREFETCH 0
#endif
__device__ __forceinline__ void leaf_test(const mcgd::SceneView& S, uint32_t first, uint32_t cnt, V3 o, V3 d,
                                          float tmin, float& closest, uint32_t& prim, float& t_out,
                                          float& b1_out, float& b2_out, bool& found) {
#if MCG_TRI_PREFETCH
    if (cnt == 0) return;
    PrimG cur = load_prim(S, first);
    for (uint32_t i = first; i < first + cnt; ++i) {
        PrimG nxt = cur;
        if (i + 1 < first + cnt) nxt = load_prim(S, i + 1);
        float t, b1, b2;
        if (hit_prim_g(cur, o, d, tmin, closest, t, b1, b2)) {
            closest = t;
            prim = i;
            t_out = t;
            b1_out = b1;
            b2_out = b2;
            found = true;
        }
        cur = nxt;
    }
#else
    for (uint32_t i = first; i < first + cnt; ++i) {
        float t, b1, b2;
        if (hit_prim(S, i, o, d, tmin, closest, t, b1, b2)) {
            closest = t;
            prim = i;
            t_out = t;
            b1_out = b1;
            b2_out = b2;
            found = true;
        }
    }
#endif
}

// The leaf phase with the warp's (ray, primitive) pairs redistributed over
// all 32 lanes (MCG_LEAF_REDIST): only ~1/3 of the lanes hold a leaf when
// the while-while loop reaches it, and each tests its <= 4 (<= 7) triangles
// one after the other. Here the warp's pairs are numbered lane by lane
// (prefix sum of the counts), each lane tests the pairs r*32 + lane against
// its owner's ray with tmax = the owner's closest before this leaf, and the
// owner then takes its results in primitive order with the reference's
// strict update (scene.cpp:252-278: closest = t iff t < closest). This is
// the sequential decision exactly: a primitive's (t, b1, b2) do not depend
// on tmax, a triangle is accepted iff t < tmax, and a sphere takes its
// nearer root below tmax -- so "hit below the old closest, then t < current
// closest" accepts exactly what "hit below the current closest" accepts,
// with the same values. Warp-collective: every lane calls it.
// Off: exact, but slower -- trace_closest 1.76 vs 1.43 ms per launch, 700 vs
// 629 ms per bench render (gpurun_out r2 ab_c: the ~26 shuffles per round
// of 32 pairs cost more than the idle lanes of the serial leaf loop).
#ifndef MCG_LEAF_REDIST
#define MCG_LEAF_REDIST 0
#endif
__device__ __forceinline__ void leaf_redist(const mcgd::SceneView& S, bool has, int32_t code, V3 o, V3 d,
                                            float tmin, float& closest, uint32_t& prim, float& t_out,
                                            float& b1_out, float& b2_out, bool& found, uint32_t& prims_tested) {
    const unsigned lane = threadIdx.x & 31u;
    uint32_t first = 0, cnt = 0;
    if (has) {
        const uint32_t v = static_cast<uint32_t>(~code);
        first = v >> 3;
        cnt = v & 7u;
    }
    uint32_t incl = cnt;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t x = __shfl_up_sync(mcgd::kFull, incl, off);
        if (lane >= static_cast<unsigned>(off)) incl += x;
    }
    const uint32_t total = __shfl_sync(mcgd::kFull, incl, 31);
    if (total == 0) return;
    const uint32_t excl = incl - cnt;
    const uint32_t maxcnt = __reduce_max_sync(mcgd::kFull, cnt);
    prims_tested += cnt;
    const float c0 = closest;
    for (uint32_t base = 0; base < total; base += 32u) {
        const uint32_t qi = base + lane;
        // owner: the first lane whose inclusive count exceeds qi
        int owner = 0;
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
            if (__shfl_sync(mcgd::kFull, incl, owner + step - 1) <= qi) owner += step;
        }
        const float ox = __shfl_sync(mcgd::kFull, o.x, owner), oy = __shfl_sync(mcgd::kFull, o.y, owner),
                    oz = __shfl_sync(mcgd::kFull, o.z, owner);
        const float dx = __shfl_sync(mcgd::kFull, d.x, owner), dy = __shfl_sync(mcgd::kFull, d.y, owner),
                    dz = __shfl_sync(mcgd::kFull, d.z, owner);
        const float tmax = __shfl_sync(mcgd::kFull, c0, owner);
        const uint32_t pi = __shfl_sync(mcgd::kFull, first, owner) + qi - __shfl_sync(mcgd::kFull, excl, owner);
        float t = __int_as_float(0x7f800000), b1 = 0.0f, b2 = 0.0f;
        if (qi < total) {
            float tt, bb1, bb2;
            if (hit_prim(S, pi, V3{ox, oy, oz}, V3{dx, dy, dz}, tmin, tmax, tt, bb1, bb2)) {
                t = tt;
                b1 = bb1;
                b2 = bb2;
            }
        }
        for (uint32_t k = 0; k < maxcnt; ++k) {
            const uint32_t g = excl + k;
            const bool mine = k < cnt && g >= base && g < base + 32u;
            const int src = mine ? static_cast<int>(g - base) : static_cast<int>(lane);
            const float kt = __shfl_sync(mcgd::kFull, t, src);
            const float kb1 = __shfl_sync(mcgd::kFull, b1, src);
            const float kb2 = __shfl_sync(mcgd::kFull, b2, src);
            if (mine && kt < closest) {
                closest = kt;
                prim = first + k;
                t_out = kt;
                b1_out = kb1;
                b2_out = kb2;
                found = true;
            }
        }
    }
}

__device__ __forceinline__ bool closest_ww4s(const mcgd::SceneView& S, bool active, V3 o, V3 d,
                                             float tmin, float tmax, uint32_t& prim, float& t_out,
                                             float& b1_out, float& b2_out, uint32_t& nodes_visited,
                                             uint32_t& prims_tested) {
    const V3 inv{1.0f / d.x, 1.0f / d.y, 1.0f / d.z};
    const RayQ rq = make_rayq(o, inv);
    int2 st[64];
    int top = 0;
    int32_t nc = 0;  // register-held next entry
    float ne = 0.0f;
    bool has_n = false;
    if (active && S.n_nodes) {
        const float4 lo = __ldg(S.nodes), hi = __ldg(S.nodes + 1);
        float E, T1;
        slab(o, inv, lo, hi, tmin, E, T1);
        if (!(T1 < E)) {
            nc = entry_code(S.root_a, S.root_b);
            ne = E;
            has_n = true;
        }
    }
    bool found = false;
    float closest = tmax;
    int32_t lc = 0;
    bool leaf = false;
#if MCG_CLOSEST_LEAVES > 1
    int32_t lc2 = 0;   // a second leaf, popped while speculating; tested
    float le2 = 0.0f;  // after the first with its cull test re-done
    bool leaf2 = false;
#endif
    while (__any_sync(mcgd::kFull, has_n || leaf)) {
        // Phase 1: pop/expand until every lane holds a leaf or is done;
        // lanes holding one keep expanding internal entries (speculation).
        for (;;) {
            // culled entries (the reference's test at pop) are skipped in a
            // tight loop rather than one per warp-wide iteration
            while (has_n && closest < ne) {
                ++nodes_visited;
                has_n = false;
                if (top > 0) {
                    --top;
                    const int2 e = st[top];
                    nc = e.x;
                    ne = __int_as_float(e.y);
                    has_n = true;
                }
            }
            if (has_n) {
                if (nc < 0) {
                    if (!leaf) {
                        ++nodes_visited;
                        leaf = true;
                        lc = nc;
                        has_n = false;
                    }
#if MCG_CLOSEST_LEAVES > 1
                    else if (!leaf2) {
                        ++nodes_visited;
                        leaf2 = true;
                        lc2 = nc;
                        le2 = ne;
                        has_n = false;
                    }
#endif
                } else {
                    ++nodes_visited;
                    has_n = false;
                    if constexpr (mcgd::kClosestWidth == 4) {
                        const float4* p = S.quads_soa + 8 * nc;
                        float E[4], T1[4];
                        box4(p, rq, tmin, E, T1);
                        const int4 ea = __ldg(reinterpret_cast<const int4*>(p + 6));
                        const int4 eb = __ldg(reinterpret_cast<const int4*>(p + 7));
                        const int32_t A[4] = {ea.x, ea.y, ea.z, ea.w}, B[4] = {eb.x, eb.y, eb.z, eb.w};
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            if (B[k] != 0 && !(T1[k] < E[k])) {
                                if (has_n) {
                                    MCG_CHECK(top < 64);
                                    st[top++] = make_int2(nc, __float_as_int(ne));
                                }
                                nc = entry_code(A[k], B[k]);
                                ne = E[k];
                                has_n = true;
                            }
                        }
                    } else {
                        const float4* p = S.quads + 2 * mcgd::kClosestWidth * nc;
#pragma unroll
                        for (int k = 0; k < mcgd::kClosestWidth; ++k) {
                            const float4 lo = __ldg(p + 2 * k), hi = __ldg(p + 2 * k + 1);
                            const int32_t eb = __float_as_int(hi.w);
                            if (eb == 0) continue;  // empty entry
                            float E, T1;
                            slab(o, inv, lo, hi, tmin, E, T1);
                            if (!(T1 < E)) {
                                if (has_n) {
                                    MCG_CHECK(top < 64);
                                    st[top++] = make_int2(nc, __float_as_int(ne));
                                }
                                nc = entry_code(__float_as_int(lo.w), eb);
                                ne = E;
                                has_n = true;
                            }
                        }
                    }
                }
            }
            if (!has_n && top > 0) {
                --top;
                const int2 e = st[top];
                nc = e.x;
                ne = __int_as_float(e.y);
                has_n = true;
            }
#ifdef MCG_PREFETCH_NODES
            // the next node's 128-byte line on its way while the warp syncs
            if (mcgd::kClosestWidth == 4 && has_n && nc >= 0) {
                asm volatile("prefetch.global.L1 [%0];" ::"l"(S.quads_soa + 8 * nc));
            }
#endif
            if (__all_sync(mcgd::kFull, leaf || !has_n)) break;
        }
        // Phase 2: every lane holding a leaf tests it (the reference's order).
#if MCG_LEAF_REDIST
        leaf_redist(S, leaf, lc, o, d, tmin, closest, prim, t_out, b1_out, b2_out, found, prims_tested);
        leaf = false;
#if MCG_CLOSEST_LEAVES > 1
        {
            // the second leaf: its cull test against the closest it would see
            const bool go2 = leaf2 && !(closest < le2);
            leaf2 = false;
            leaf_redist(S, go2, lc2, o, d, tmin, closest, prim, t_out, b1_out, b2_out, found, prims_tested);
        }
#endif
        if (false) {
#else
        if (leaf) {
#endif
            const uint32_t v = static_cast<uint32_t>(~lc);
            const uint32_t first = v >> 3, cnt = v & 7u;
            prims_tested += cnt;
            leaf_test(S, first, cnt, o, d, tmin, closest, prim, t_out, b1_out, b2_out, found);
            leaf = false;
#if MCG_CLOSEST_LEAVES > 1
            if (leaf2) {
                leaf2 = false;
                if (!(closest < le2)) {  // its cull test, against the closest it would see
                    const uint32_t v2 = static_cast<uint32_t>(~lc2);
                    const uint32_t first2 = v2 >> 3, cnt2 = v2 & 7u;
                    prims_tested += cnt2;
                    leaf_test(S, first2, cnt2, o, d, tmin, closest, prim, t_out, b1_out, b2_out, found);
                }
            }
#endif
        }
    }
    return found;
}


// Any hit over a kW-wide tree (the SAH shadow tree over the reference's
// leaves): speculative while-while like closest_ww4s; of the entries a node
// passes, the nearest stays in registers (popped next), the rest go to the
// stack in entry order -- any order is exact for a boolean query.
#ifndef MCG_SHADOW_LEAVES
#define MCG_SHADOW_LEAVES 1
#endif
template <int kW, int kLeaves = MCG_SHADOW_LEAVES>
__device__ __forceinline__ bool any_wws(const float4* Q, int32_t root_a, int32_t root_b, const mcgd::SceneView& S,
                                        bool active, V3 o, V3 d, float tmin, float tmax,
                                        uint32_t& nodes_visited, uint32_t& prims_tested,
                                        const float4* Qs = nullptr) {
    const V3 inv{1.0f / d.x, 1.0f / d.y, 1.0f / d.z};
    const RayQ rq = make_rayq(o, inv);
    int32_t st[64];
    int top = 0;
    int32_t nc = 0;
    bool has_n = false;
    if (active && S.n_nodes) {
        const float4 lo = __ldg(S.nodes), hi = __ldg(S.nodes + 1);
        float E, T1;
        slab(o, inv, lo, hi, tmin, E, T1);
        if (!(fminf(tmax, T1) < E)) {
            nc = entry_code(root_a, root_b);
            has_n = true;
        }
    }
    bool hit = false;
    int32_t lc = 0, lc2 = 0;
    bool leaf = false, leaf2 = false;
    while (__any_sync(mcgd::kFull, has_n || leaf)) {
        for (;;) {
            if (has_n) {
                if (nc < 0) {
                    if (!leaf) {
                        ++nodes_visited;
                        leaf = true;
                        lc = nc;
                        has_n = false;
                    } else if (kLeaves > 1 && !leaf2) {
                        ++nodes_visited;
                        leaf2 = true;
                        lc2 = nc;
                        has_n = false;
                    }
                } else {
                    ++nodes_visited;
                    has_n = false;
                    float best = __int_as_float(0x7f800000);
                    if (kW == 4 && Qs != nullptr) {
                        // transposed node: four boxes with packed arithmetic
                        const float4* p = Qs + 8 * nc;
                        float E[4], T1[4];
                        box4(p, rq, tmin, E, T1);
                        const int4 ea = __ldg(reinterpret_cast<const int4*>(p + 6));
                        const int4 eb = __ldg(reinterpret_cast<const int4*>(p + 7));
                        const int32_t A[4] = {ea.x, ea.y, ea.z, ea.w}, B[4] = {eb.x, eb.y, eb.z, eb.w};
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            if (B[k] != 0 && !(fminf(tmax, T1[k]) < E[k])) {
                                const int32_t code = entry_code(A[k], B[k]);
                                if (!has_n) {
                                    nc = code;
                                    best = E[k];
                                    has_n = true;
                                } else if (E[k] < best) {
                                    MCG_CHECK(top < 64);
                                    st[top++] = nc;
                                    nc = code;
                                    best = E[k];
                                } else {
                                    MCG_CHECK(top < 64);
                                    st[top++] = code;
                                }
                            }
                        }
                    } else {
                    const float4* p = Q + 2 * kW * nc;
#pragma unroll
                    for (int k = 0; k < kW; ++k) {
                        const float4 lo = __ldg(p + 2 * k), hi = __ldg(p + 2 * k + 1);
                        const int32_t eb = __float_as_int(hi.w);
                        if (eb == 0) break;  // entries are packed: the first empty ends the node
                        float E, T1;
                        slab(o, inv, lo, hi, tmin, E, T1);
                        if (!(fminf(tmax, T1) < E)) {
                            const int32_t code = entry_code(__float_as_int(lo.w), eb);
                            if (!has_n) {
                                nc = code;
                                best = E;
                                has_n = true;
                            } else if (E < best) {
                                MCG_CHECK(top < 64);
                                    st[top++] = nc;
                                nc = code;
                                best = E;
                            } else {
                                MCG_CHECK(top < 64);
                                    st[top++] = code;
                            }
                        }
                    }
                    }
                }
            }
            if (!has_n && top > 0) {
                nc = st[--top];
                has_n = true;
            }
            if (__all_sync(mcgd::kFull, leaf || !has_n)) break;
        }
        if (leaf) {
#pragma unroll
            for (int l = 0; l < kLeaves; ++l) {
                if (l == 1 && (!leaf2 || hit)) break;
                const uint32_t v = static_cast<uint32_t>(~(l == 0 ? lc : lc2));
                const uint32_t first = v >> 3, cnt = v & 7u;
                prims_tested += cnt;
                for (uint32_t i = first; i < first + cnt; ++i) {
                    float t, b1, b2;
                    if (hit_prim(S, i, o, d, tmin, tmax, t, b1, b2)) {
                        hit = true;
                        break;
                    }
                }
            }
            leaf = false;
            leaf2 = false;
            if (hit) has_n = false, top = 0;
        }
    }
    return hit;
}

// ---------------------------------------------------------------------------
// Packet traversal: the warp walks the 4-wide tree together, one entry at a
// time, each entry carrying the mask of lanes that pushed it. The
// reference's visit order does not depend on the ray (its DFS always pushes
// left then right, scene.cpp:259-272), so every lane still sees its own
// entries in its own LIFO order -- the packet stack is the interleaving of
// 32 identical-order private stacks -- and each lane makes exactly its own
// decisions: the ray-only half of a box test when the entry is pushed, the
// closest-dependent half (closest < E, per lane, E kept in shared memory)
// when it is popped. Pops and pushes are warp-uniform, so the stack costs
// one shared-memory word pair per entry instead of per lane, and the box
// tests run with every interested lane converged. Coherent rays (primary
// rays, shadow rays toward one light from Morton-sorted points) share most
// of their entries; the price is that a lane waits through entries that
// only other lanes need.
// Per-warp shared memory: code[D], mask[D] (+ E[D][32] for closest hit).
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool closest_pk(const mcgd::SceneView& S, bool active, V3 o, V3 d, float tmin,
                                           float tmax, uint32_t& prim, float& t_out, float& b1_out,
                                           float& b2_out, uint32_t& nodes_visited, uint32_t& prims_tested,
                                           int32_t* s_code, uint32_t* s_mask, float* s_e) {
    const uint32_t lane = threadIdx.x & 31u;
    const V3 inv{1.0f / d.x, 1.0f / d.y, 1.0f / d.z};
    int top = 0;
    if (S.n_nodes) {
        bool ok = false;
        float E = 0.0f, T1 = 0.0f;
        if (active) {
            slab(o, inv, __ldg(S.nodes), __ldg(S.nodes + 1), tmin, E, T1);
            ok = !(T1 < E);
        }
        const uint32_t m = __ballot_sync(mcgd::kFull, ok);
        if (m) {
            if (lane == 0) {
                s_code[0] = entry_code(S.root_a, S.root_b);
                s_mask[0] = m;
            }
            s_e[lane] = E;
            top = 1;
        }
    }
    __syncwarp();
    bool found = false;
    float closest = tmax;
    while (top > 0) {
        --top;
        const int32_t code = s_code[top];
        const uint32_t m = s_mask[top];
        bool me = (m >> lane) & 1u;
        if (me) {
            ++nodes_visited;
            if (closest < s_e[top * 32 + lane]) me = false;  // the reference's test at pop
        }
        if (__ballot_sync(mcgd::kFull, me) == 0u) {
            __syncwarp();
            continue;
        }
        if (code < 0) {
            if (me) {
                const uint32_t v = static_cast<uint32_t>(~code);
                const uint32_t first = v >> 3, cnt = v & 7u;
                prims_tested += cnt;
                for (uint32_t i = first; i < first + cnt; ++i) {
                    float t, b1, b2;
                    if (hit_prim(S, i, o, d, tmin, closest, t, b1, b2)) {
                        closest = t;
                        prim = i;
                        t_out = t;
                        b1_out = b1;
                        b2_out = b2;
                        found = true;
                    }
                }
            }
        } else {
            const float4* p = S.quads + 2 * mcgd::kClosestWidth * code;
#pragma unroll
            for (int k = 0; k < mcgd::kClosestWidth; ++k) {
                const float4 lo = __ldg(p + 2 * k), hi = __ldg(p + 2 * k + 1);
                const int32_t eb = __float_as_int(hi.w);
                if (eb == 0) continue;  // empty entry (uniform)
                float E, T1;
                slab(o, inv, lo, hi, tmin, E, T1);
                const uint32_t mk = __ballot_sync(mcgd::kFull, me && !(T1 < E));
                if (mk) {
                    if (lane == 0) {
                        s_code[top] = entry_code(__float_as_int(lo.w), eb);
                        s_mask[top] = mk;
                    }
                    s_e[top * 32 + lane] = E;
                    ++top;
                }
            }
        }
        __syncwarp();
    }
    return found;
}

__device__ __forceinline__ bool any_pk(const mcgd::SceneView& S, bool active, V3 o, V3 d, float tmin,
                                       float tmax, uint32_t& nodes_visited, uint32_t& prims_tested,
                                       int32_t* s_code, uint32_t* s_mask) {
    const uint32_t lane = threadIdx.x & 31u;
    const V3 inv{1.0f / d.x, 1.0f / d.y, 1.0f / d.z};
    int top = 0;
    if (S.n_nodes) {
        bool ok = false;
        if (active) {
            float E, T1;
            slab(o, inv, __ldg(S.nodes), __ldg(S.nodes + 1), tmin, E, T1);
            ok = !(fminf(tmax, T1) < E);
        }
        const uint32_t m = __ballot_sync(mcgd::kFull, ok);
        if (m) {
            if (lane == 0) {
                s_code[0] = entry_code(S.root_a, S.root_b);
                s_mask[0] = m;
            }
            top = 1;
        }
    }
    __syncwarp();
    bool hit = false;
    while (top > 0) {
        --top;
        const int32_t code = s_code[top];
        const uint32_t m = s_mask[top] & ~__ballot_sync(mcgd::kFull, hit);
        if (m == 0u) {
            __syncwarp();
            continue;
        }
        const bool me = (m >> lane) & 1u;
        if (me) ++nodes_visited;
        if (code < 0) {
            if (me) {
                const uint32_t v = static_cast<uint32_t>(~code);
                const uint32_t first = v >> 3, cnt = v & 7u;
                prims_tested += cnt;
                for (uint32_t i = first; i < first + cnt; ++i) {
                    float t, b1, b2;
                    if (hit_prim(S, i, o, d, tmin, tmax, t, b1, b2)) {
                        hit = true;
                        break;
                    }
                }
            }
            if (__all_sync(mcgd::kFull, hit || !active)) break;
        } else {
            const float4* p = S.quads + 2 * mcgd::kClosestWidth * code;
#pragma unroll
            for (int k = 0; k < mcgd::kClosestWidth; ++k) {
                const float4 lo = __ldg(p + 2 * k), hi = __ldg(p + 2 * k + 1);
                const int32_t eb = __float_as_int(hi.w);
                if (eb == 0) break;  // uniform
                float E, T1;
                slab(o, inv, lo, hi, tmin, E, T1);
                const uint32_t mk = __ballot_sync(mcgd::kFull, me && !(fminf(tmax, T1) < E));
                if (mk) {  // uniform; entry order (any order is exact for a boolean query)
                    if (lane == 0) {
                        s_code[top] = entry_code(__float_as_int(lo.w), eb);
                        s_mask[top] = mk;
                    }
                    ++top;
                }
            }

        }
        __syncwarp();
    }
    return hit;
}

// Per-warp packet stacks in dynamic shared memory (depth D entries).
__device__ __forceinline__ void pk_stacks(int depth, bool closest, int32_t*& code, uint32_t*& mask,
                                          float*& e) {
    extern __shared__ float pk_smem[];
    const uint32_t w = threadIdx.x >> 5;
    const size_t per_warp = static_cast<size_t>(depth) * (closest ? 2 + 32 : 2);
    float* base = pk_smem + w * per_warp;
    code = reinterpret_cast<int32_t*>(base);
    mask = reinterpret_cast<uint32_t*>(base + depth);
    e = base + 2 * depth;
}

// Pass start: primary rays of every path of the pass, traced to vertex 0,
// state written at layout position = path id.
#ifndef MCG_PRIMARY_BLOCK
#define MCG_PRIMARY_BLOCK 128
#endif
template <uint32_t kMax>
__global__ void __launch_bounds__(MCG_PRIMARY_BLOCK) k_primary(RenderView R) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t nvis = 0, ntest = 0;
    const bool active = i < R.n_paths;
    V3 o{0.0f, 0.0f, 0.0f}, d{1.0f, 1.0f, 1.0f};
    if (active) {
        const uint32_t slot_j = i / R.n_pix;
        const uint32_t pixel = R.pix[i - slot_j * R.n_pix];
        const uint64_t rkey = mcgd::path_key(R.seed, pixel, R.sample0 + slot_j);
        camera_ray(R, pixel, rkey, o, d);
    }
    uint32_t prim = 0;
    float t = 0.0f, b1 = 0.0f, b2 = 0.0f;
    const bool found = closest_ww4s(R.S, active, o, d, kTMin, __int_as_float(0x7f800000), prim, t, b1, b2,
                                    nvis, ntest);
    if (active) {
        const float4 ro0 = make_float4(o.x, o.y, o.z, 0.0f);
        float4 ro = ro0;
        const float4 rd = make_float4(d.x, d.y, d.z, R.cam[11]);
        const float4 thr = make_float4(1.0f, 1.0f, 1.0f, __uint_as_float(0u));
        const float4 L = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        const uint32_t key = hit_record<kMax>(R, i, i, ro, rd, thr, L, found, prim, t, b1, b2, 0);
        R.pa[i].ro = ro0;   // the width at the origin (the shade propagates it)
        R.pa[i].rd = rd;
        R.pb[i] = PathVal{thr, make_float4(0.0f, 0.0f, 0.0f, __uint_as_float(i))};
        R.keys[i] = key;
        R.vals[i] = i;
    }
    mcgd::warp_add(R.stats + kStatNodes, nvis);
    mcgd::warp_add(R.stats + kStatPrims, ntest);
}

// ---------------------------------------------------------------------------
// Scene queries for a batch of rays (Scene::intersect / Scene::occluded,
// scene.cpp:252-298) through any of the traversal variants the renderer
// uses -- the parity tests check each one against the oracle's DFS.
// variant: 0 per-thread binary DFS, 1 while-while child pairs, 2 4-wide,
// 3 speculative 4-wide (the default of render()).
// ---------------------------------------------------------------------------
template <int kVar>
__global__ void __launch_bounds__(256) k_intersect_batch(mcgd::SceneView S, const float* rays, uint32_t n,
                                                         float tmin, float tmax, float* out, int depth) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    const bool active = i < n;
    V3 o{0.0f, 0.0f, 0.0f}, d{1.0f, 1.0f, 1.0f};
    if (active) {
        o = V3{rays[6 * i], rays[6 * i + 1], rays[6 * i + 2]};
        d = V3{rays[6 * i + 3], rays[6 * i + 4], rays[6 * i + 5]};
    }
    uint32_t prim = 0, nv = 0, nt = 0;
    float t = 0.0f, b1 = 0.0f, b2 = 0.0f;
    bool found;
    if (kVar == 0) found = active && traverse_closest(S, o, d, tmin, tmax, prim, t, b1, b2, nv, nt);
    else if (kVar == 1) found = closest_ww(S, active, o, d, tmin, tmax, prim, t, b1, b2, nv, nt);
    else if (kVar == 2) found = closest_ww4(S, active, o, d, tmin, tmax, prim, t, b1, b2, nv, nt);
    else if (kVar == 3) found = closest_ww4s(S, active, o, d, tmin, tmax, prim, t, b1, b2, nv, nt);
    else {
        int32_t* pc;
        uint32_t* pm;
        float* pe;
        pk_stacks(depth, true, pc, pm, pe);
        found = closest_pk(S, active, o, d, tmin, tmax, prim, t, b1, b2, nv, nt, pc, pm, pe);
    }
    if (!active) return;
    float* w = out + 24ull * i;
    float v[24] = {};
    if (found) {
        const Surface sf = surface(S, o, d, prim, t, b1, b2);
        const float vals[21] = {1.0f, t, sf.p.x, sf.p.y, sf.p.z, sf.n.x, sf.n.y, sf.n.z, sf.u, sf.v,
                                static_cast<float>(sf.slot), sf.e1.x, sf.e1.y, sf.e1.z, sf.e2.x, sf.e2.y,
                                sf.e2.z, sf.d1.x, sf.d1.y, sf.d2.x, sf.d2.y};
#pragma unroll
        for (int k = 0; k < 21; ++k) v[k] = vals[k];
    }
#pragma unroll
    for (int k = 0; k < 24; ++k) w[k] = v[k];
}

template <int kVar>
__global__ void __launch_bounds__(256) k_occluded_batch(mcgd::SceneView S, const float* rays, uint32_t n,
                                                        float tmin, const float* tmax, uint8_t* out, int depth) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    const bool active = i < n;
    V3 o{0.0f, 0.0f, 0.0f}, d{1.0f, 1.0f, 1.0f};
    float tm = 0.0f;
    if (active) {
        o = V3{rays[6 * i], rays[6 * i + 1], rays[6 * i + 2]};
        d = V3{rays[6 * i + 3], rays[6 * i + 4], rays[6 * i + 5]};
        tm = tmax[i];
    }
    uint32_t nv = 0, nt = 0;
    bool occ;
    if (kVar == 0) occ = active && traverse_any(S, o, d, tmin, tm, nv, nt);
    else if (kVar == 1) occ = any_ww(S, active, o, d, tmin, tm, nv, nt);
    else if (kVar == 2) occ = any_ww4(S, active, o, d, tmin, tm, nv, nt);
    else if (kVar == 3) occ = any_wws<mcgd::kClosestWidth>(S.quads, S.root_a, S.root_b, S, active, o, d, tmin, tm, nv, nt, S.quads_soa);
    else if (kVar == 5) occ = any_wws<mcgd::kShadowWidth>(S.squads, S.sroot_a, S.sroot_b, S, active, o, d, tmin, tm, nv, nt, S.squads_soa);
    else {
        int32_t* pc;
        uint32_t* pm;
        float* pe;
        pk_stacks(depth, false, pc, pm, pe);
        occ = any_pk(S, active, o, d, tmin, tm, nv, nt, pc, pm);
    }
    if (active) out[i] = occ ? 1 : 0;
}

// Shadow rays, one per thread over the queue, speculative 4-wide traversal
// of the SAH tree over the reference's leaves (kSah) or of the reference's
// own tree.
#ifndef MCG_TRACE_MINB
#define MCG_TRACE_MINB 8
#endif
template <bool kSah>
#ifndef MCG_SHADOW_BLOCK
#define MCG_SHADOW_BLOCK 128
#endif
#ifndef MCG_SHADOW_MINB
#define MCG_SHADOW_MINB 10
#endif
__global__ void __launch_bounds__(MCG_SHADOW_BLOCK, MCG_SHADOW_MINB) k_shadow_ww(RenderView R) {
    const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t nvis = 0, ntest = 0;
    const bool active = q < *R.shadow_count;
    uint32_t s = 0;
    V3 o{0.0f, 0.0f, 0.0f}, d{1.0f, 1.0f, 1.0f};
    float tmax = 0.0f;
    if (active) {
        s = R.squeue[q];
        const float4 so = R.sro[s], sd = R.srd[s];
        o = V3{so.x, so.y, so.z};
        d = V3{sd.x, sd.y, sd.z};
        tmax = so.w;
    }
    const bool occ = kSah ? any_wws<mcgd::kShadowWidth>(R.S.squads, R.S.sroot_a, R.S.sroot_b, R.S, active, o, d, kTMin, tmax, nvis, ntest, R.S.squads_soa)
                          : any_wws<mcgd::kClosestWidth>(R.S.quads, R.S.root_a, R.S.root_b, R.S, active, o, d, kTMin, tmax, nvis, ntest, R.S.quads_soa);
    if (active) R.vis[s] = occ ? 0 : 1;
    mcgd::warp_add(R.stats + kStatOccluded, active && occ ? 1u : 0u);
    mcgd::warp_add(R.stats + kStatShadow, active ? 1u : 0u);
    mcgd::warp_add(R.stats + kStatNodesShadow, nvis);
    mcgd::warp_add(R.stats + kStatPrimsShadow, ntest);
}

// Closest hits of the continuation rays, one per thread at its own layout
// position, speculative 4-wide traversal in the reference's order.
#ifndef MCG_TRACE_BLOCK
#define MCG_TRACE_BLOCK 128
#endif
template <uint32_t kMax>
__global__ void __launch_bounds__(MCG_TRACE_BLOCK, MCG_TRACE_MINB) k_trace_closest_ww(RenderView R, const uint32_t* count, int vtx) {
    const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t nvis = 0, ntest = 0;
    const bool active = q < *count;
    float4 ro{}, rd{};
    if (active) {
        ro = R.pa[q].ro;
        rd = R.pa[q].rd;
    }
    const V3 o{ro.x, ro.y, ro.z}, d = active ? V3{rd.x, rd.y, rd.z} : V3{1.0f, 1.0f, 1.0f};
    uint32_t prim = 0;
    float t = 0.0f, b1 = 0.0f, b2 = 0.0f;
    const bool found = closest_ww4s(R.S, active, o, d, kTMin, __int_as_float(0x7f800000), prim, t, b1, b2,
                                    nvis, ntest);
    if (active) {
        const uint32_t pid = __float_as_uint(R.pb[q].L.w);
        uint32_t key;
        if (found) {
            key = hit_record<kMax>(R, q, pid, ro, rd, make_float4(0, 0, 0, 0), make_float4(0, 0, 0, 0), true, prim, t,
                             b1, b2, vtx);
        } else {
            // the path ends; k_resolve_lights (which runs after this kernel
            // and the shadow rays) adds throughput * env to its final radiance
            key = no_hit_key(R);
        }
        R.keys[q] = key;
        R.vals[q] = q;
    }
    mcgd::warp_add(R.stats + kStatClosestRays, active ? 1u : 0u);
    mcgd::warp_add(R.stats + kStatNodes, nvis);
    mcgd::warp_add(R.stats + kStatPrims, ntest);
}

// Look-ahead probe of every live hit, before the material sort: the shading
// point is rebuilt from the hit record exactly as k_shade will (shade_input),
// the descriptors of the material's first kAhead cache points are built and
// probed (cache.cpp:121-136), and the hit bits enter the sort key below the
// material slot -- so the shade sees warps whose lanes all hit (the group
// skips the subtree, Alg. 2) or all miss (the subtree runs with every lane
// active), instead of a few misses holding a whole warp in the subtree.
// Concurrent mode: a lookup observed before the vertex's stores is one of the
// interleavings the reference's threads allow (slots are write-once, a hit
// stays valid). Deterministic mode: the probe runs after the previous epoch's
// ordered apply, so it reads the epoch-start table -- the same rule.
__global__ void __launch_bounds__(256) k_lookahead(RenderView R, const uint32_t* count) {
    const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= (count ? *count : R.n_paths)) return;
    const uint32_t key = R.keys[q];
    if (key_slot(R, key) >= R.S.n_programs) return;
    const PathRay& pr = R.pa[q];
    const mcgd::ShadeIn in = shade_input(pr.rd, pr.sp0, pr.sp1, pr.sp2, pr.sp3);
    R.keys[q] = look_ahead<mcgd::kAhead>(R, q, key, in);
}

// Finishes vertex b at sorted position i, after the shadow rays and the
// continuation rays of the vertex: adds the visible light contributions in
// light order (the oracle's summation order); the path ends (fin[pid]) at the
// last vertex, or with the environment term when its continuation ray missed.
// Writes "no hit" sort keys for the slots past the live list.
__global__ void __launch_bounds__(256) k_resolve_lights(RenderView R, int b) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= R.n_paths) return;
    const uint32_t slot = key_slot(R, R.skey[i]);
    const bool live = slot < R.S.n_programs;
    if (live) {
        const uint32_t nl = R.S.n_plights + R.S.n_rlights;
        const PathVal pv = R.pb[i];
        float4 L = pv.L;
        const uint32_t pid = __float_as_uint(pv.L.w);
        for (uint32_t j = 0; j < nl; ++j) {
            const uint32_t s = i * nl + j;
            const float4 c = R.scon[s];
            if (c.w != 0.0f && R.vis[s]) {
                L.x = L.x + c.x;
                L.y = L.y + c.y;
                L.z = L.z + c.z;
            }
        }
        if (b >= R.max_bounces) {
            R.fin[pid] = make_float4(L.x, L.y, L.z, pv.thr.w);
        } else if (R.keys[i] == no_hit_key(R)) {
            // the continuation ray missed (k_trace_closest_ww): env term, path ends
            const float4 thr = pv.thr;
            R.fin[pid] = make_float4(L.x + thr.x * R.S.env[0], L.y + thr.y * R.S.env[1],
                                          L.z + thr.z * R.S.env[2], thr.w);
        } else {
            R.pb[i].L = L;
        }
    } else {
        R.keys[i] = no_hit_key(R);
        R.vals[i] = i;
    }
}


// Material evaluation of every live hit, in sorted (material, Morton)
// order, then NEE and the bounce; the path's state moves from its old layout
// position q = order[i] to i in the next layout.
// (256, 3): 80 registers (a few spill slots), three resident blocks. With
// the look-ahead sort the subtrees run with full warps and the kernel is
// bound by dependent-latency stalls, so resident warps pay; 256-thread
// blocks halve the blocks that stage their programs' bytecode. Measured per
// bench render: (128, 4) 795.7 ms, (128, 5) 784.7 -> 767.8 on later builds,
// (256, 3) 764.5, (256, 5: 48 registers, 824 bytes of spills) 764.5,
// (128, 8 / 10) 801.1 / 788.4.
#ifndef MCG_SHADE_MINB
#define MCG_SHADE_MINB 3
#endif
template <bool kDeferred, bool kSmemCode>
#ifndef MCG_SHADE_BLOCK
#define MCG_SHADE_BLOCK 256
#endif
__global__ void __launch_bounds__(MCG_SHADE_BLOCK, MCG_SHADE_MINB) k_shade(RenderView R, const uint32_t* __restrict__ skey,
                                               const uint32_t* __restrict__ order, int max_stack,
                                               uint32_t wh, int b) {
    extern __shared__ float smem[];
    __shared__ uint8_t s_perm[256];
    __shared__ uint32_t s_code_lo, s_code_hi;
    mcgd::stage_perm(s_perm);
    // Blocks visit the sorted list in a scattered order (concurrent mode):
    // the paths of one texel are contiguous there (Morton order), and the
    // first block to store wins the texel -- in sorted order that would be
    // the path at the texel's spatial corner every time, a biased first
    // insert (larger cached-vs-uncached error than the reference's threads).
    const uint32_t blk = static_cast<uint32_t>((static_cast<uint64_t>(blockIdx.x) * R.shade_perm) % gridDim.x);
    const uint32_t i = blk * blockDim.x + threadIdx.x;
    const uint32_t slot = i < R.n_paths ? key_slot(R, skey[i]) : R.S.n_programs;
    // The bytecode of the block's programs (its sorted paths span one or a
    // few material slots), after the operand stack (north_star: node bytecode
    // in shared memory).
    uint4* s_code = reinterpret_cast<uint4*>(smem + 3 * max_stack * blockDim.x);
    if (kSmemCode) {
        if (threadIdx.x == 0) {
            const uint32_t n_prog = R.S.n_programs;
            const uint32_t first = blk * blockDim.x;
            const uint32_t last = min(first + blockDim.x, R.n_paths) - 1u;
            const uint32_t s0 = first < R.n_paths ? key_slot(R, skey[first]) : n_prog;
            const uint32_t s1 = min(key_slot(R, skey[last]), n_prog - 1u);
            uint32_t lo = 0xffffffffu, hi = 0u;
            for (uint32_t sl = s0; sl <= s1 && sl < n_prog; ++sl) {
                const mcg_program pg = R.S.programs[sl];
                lo = min(lo, pg.code_offset);
                hi = max(hi, pg.code_offset + pg.code_len);
            }
            s_code_lo = lo > hi ? 0u : lo;
            s_code_hi = hi;
        }
        __syncthreads();
        const uint4* g = reinterpret_cast<const uint4*>(R.S.code);
        const uint32_t lo = s_code_lo, hi = s_code_hi;
        for (uint32_t k = lo + threadIdx.x; k < hi; k += blockDim.x) s_code[k - lo] = __ldg(g + k);
    }
    __syncthreads();
    const bool valid = slot < R.S.n_programs;
    const unsigned live = __ballot_sync(mcgd::kFull, valid);
    if (!valid) return;
    // live-path count (hits sort first): the last live position writes it
    if (i + 1 == R.n_paths || key_slot(R, skey[i + 1]) >= R.S.n_programs) R.shadow_count[2] = i + 1;
#ifdef MCG_EXP_SHADE_NOGATHER
    const uint32_t q = i;   // timing experiment only: no permutation (wrong images)
#else
    const uint32_t q = order[i];
    MCG_CHECK(q < R.n_paths);
#endif
    const unsigned grp = __match_any_sync(live, slot);
    const PathRay& pr = R.pa[q];
    const float4 rd = pr.rd, sp0 = pr.sp0, sp1 = pr.sp1, sp2 = pr.sp2, sp3 = pr.sp3;
    const PathVal pv = R.pb[q];
    const uint32_t pid = __float_as_uint(pv.L.w);
    MCG_CHECK(pid < R.n_paths);
    // the rest of the path's state is loaded now, in the same round trip as
    // the hit record, not after the VM; what the VM does not change is
    // written to the next layout right away, so little of it stays live
    float4 thr = pv.thr;
    R.pb2[i].L = pv.L;
    const mcgd::ShadeIn in = shade_input(rd, sp0, sp1, sp2, sp3);
    mcgd::Stack st{smem, smem + max_stack * blockDim.x, smem + 2 * max_stack * blockDim.x,
                   static_cast<int>(blockDim.x), static_cast<int>(threadIdx.x), max_stack};
    const uint32_t slot_j = pid / R.n_pix;
    const uint32_t pixel = __float_as_uint(sp1.w);
    const uint32_t okey = (slot_j * wh + pixel) << 6;
    mcgd::VmCounters cnt;
    const mcgd::Ahead ah{__float_as_uint(sp3.z), pr.ahead, R.ahead_on != 0};
    const mcgd::VmResult r = mcgd::run_program<kDeferred, kSmemCode>(R.S, R.C, R.cache_on != 0, R.mip_offset,
                                                                     slot, in, grp, st, s_perm, okey, R.q, cnt, ah,
                                                                     s_code, kSmemCode ? s_code_lo : 0u);
    thr.w = __uint_as_float(__float_as_uint(thr.w) + cnt.hits);
    nee_bounce(R, i, pid, pixel, b, V3{in.px, in.py, in.pz}, V3{in.nx, in.ny, in.nz}, r.value, thr, sp0.w, rd.w);
    mcgd::warp_add(R.stats + kStatLookups, cnt.lookups);
    mcgd::warp_add(R.stats + kStatHits, cnt.hits);
    mcgd::warp_add(R.stats + kStatWon, cnt.won);
    mcgd::warp_add(R.stats + kStatFull, cnt.full);
    mcgd::warp_add(R.stats + kStatStores, cnt.stores);
    mcgd::warp_add(R.stats + kStatInstrs, cnt.instrs);
    mcgd::warp_add(R.stats + kStatShade, 1u);
    mcgd::warp_add(R.stats + kStatTex, cnt.tex);
}

// Adds the finished pass into the framebuffers, samples in order, so the
// double accumulators see exactly the oracle's summation order.
__global__ void __launch_bounds__(256) k_accumulate(RenderView R, uint32_t k) {
    __shared__ unsigned long long s_hits[32];
    if (threadIdx.x < 32) s_hits[threadIdx.x] = 0ull;
    __syncthreads();
    const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q < R.n_pix) {
        const uint32_t pixel = R.pix[q];
        double r = R.radiance[3ull * pixel], g = R.radiance[3ull * pixel + 1],
               bl = R.radiance[3ull * pixel + 2], nf = R.nodes_found[pixel];
        for (uint32_t j = 0; j < k; ++j) {
            const float4 L = R.fin[j * R.n_pix + q];
            const uint32_t nodes = __float_as_uint(L.w);
            r += static_cast<double>(L.x);
            g += static_cast<double>(L.y);
            bl += static_cast<double>(L.z);
            nf += static_cast<double>(nodes);
            // hits_per_sample: one shared atomic per warp, one global per block.
            const unsigned m = __activemask();
            const uint32_t wsum = __reduce_add_sync(m, nodes);
            if ((threadIdx.x & 31u) == static_cast<unsigned>(__ffs(m) - 1) && wsum && j < 32) {
                atomicAdd(&s_hits[j], static_cast<unsigned long long>(wsum));
            }
        }
        R.radiance[3ull * pixel] = r;
        R.radiance[3ull * pixel + 1] = g;
        R.radiance[3ull * pixel + 2] = bl;
        R.nodes_found[pixel] = nf;
        R.samples[pixel] += k;
    }
    __syncthreads();
    if (R.hps && threadIdx.x < k && threadIdx.x < 32 && s_hits[threadIdx.x]) {
        atomicAdd(R.hps + R.hps_base + threadIdx.x, s_hits[threadIdx.x]);
    }
}

// An integer near frac * n that is coprime to n (b -> b * m mod n is then a
// permutation of [0, n)).
uint32_t coprime_near(uint32_t n, double frac) {
    if (n <= 2) return 1u;
    uint32_t m = std::max<uint32_t>(1u, static_cast<uint32_t>(n * frac)) | 1u;
    auto gcd = [](uint32_t a, uint32_t b) { while (b) { const uint32_t t = a % b; a = b; b = t; } return a; };
    while (gcd(m, n) != 1u) m += 2u;
    return m % n ? m % n : 1u;
}

// cache counters [lookups, hits, inserts won, lost to full cells] += the
// render's (kStat* order: lookups, hits, won, full)
__global__ void k_add_counters(unsigned long long* ctr, const unsigned long long* stats) {
    if (threadIdx.x < 4) ctr[threadIdx.x] += stats[threadIdx.x];
}

bool tile_mine(const mcg_render_params& p, int tile, int n_tiles) {
    if (p.shard_count <= 1) return true;
    if (p.shard_mode == MCG_SHARD_INTERLEAVED) return tile % p.shard_count == p.shard_rank;
    const int lo = static_cast<int>(static_cast<int64_t>(n_tiles) * p.shard_rank / p.shard_count);
    const int hi = static_cast<int>(static_cast<int64_t>(n_tiles) * (p.shard_rank + 1) / p.shard_count);
    return tile >= lo && tile < hi;
}

// Packet kernels may need more than the default 48 KB of dynamic shared memory.
void pk_smem_attr(size_t bytes) {
    const int b = static_cast<int>(bytes);
    cudaFuncSetAttribute(k_intersect_batch<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
    cudaFuncSetAttribute(k_occluded_batch<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
}

#ifndef MCG_DEFAULT_LANES
#define MCG_DEFAULT_LANES 2
#endif
constexpr int kDefaultLanes = MCG_DEFAULT_LANES;

void render_device(mcg_ctx* ctx, const mcg_render_params& P, mcg_cache* external,
                   double* d_rad, double* d_nodes, uint32_t* d_samples, mcg_render_stats* stats) {
    const DeviceScene& D = ctx->scene;
    if (!D.loaded) fail(MCG_ERR_INVALID_ARGUMENT, "no scene uploaded");
    const int W = P.width ? P.width : D.cam.cam_width;
    const int H = P.height ? P.height : D.cam.cam_height;
    if (W <= 0 || H <= 0) fail(MCG_ERR_INVALID_ARGUMENT, "image size must be positive");
    if (P.spp < 1) fail(MCG_ERR_INVALID_ARGUMENT, "spp must be >= 1");
    if (P.max_bounces < 0) fail(MCG_ERR_INVALID_ARGUMENT, "max_bounces must be >= 0");
    if (D.view.n_rlights > 31) fail(MCG_ERR_INVALID_ARGUMENT, "at most 31 rect lights");
    if (P.shard_count > 1 && (P.shard_rank < 0 || P.shard_rank >= P.shard_count)) {
        fail(MCG_ERR_INVALID_ARGUMENT, "shard_rank out of range");
    }
    const auto t0 = std::chrono::steady_clock::now();
    const uint64_t launches0 = ctx->launches;
    const bool cache_on = P.cache_mode != MCG_CACHE_OFF;
    const bool deferred = P.cache_mode == MCG_CACHE_DETERMINISTIC;
    const char* sc_env = std::getenv("MCG_SHADE_SCATTER");
    const bool scatter = !(sc_env && std::string(sc_env) == "0");
    const char* la_env = std::getenv("MCG_LOOKAHEAD");
    const bool look_ahead_req = cache_on && D.max_cache_points > 0 && D.view.ahead_cp &&
                                !(la_env && std::string(la_env) == "0");

    // Shard pixel list (16x16 tiles, tracer.hpp:19), built on the host and
    // uploaded once per (size, tiling, shard): a render call otherwise left
    // the GPU idle for the few ms this loop and copy take.
    const int ts = P.tile_size > 0 ? P.tile_size : 16;
    const int64_t pkey[6] = {W, H, ts, P.shard_count > 1 ? P.shard_rank : 0, std::max(1, P.shard_count),
                             P.shard_count > 1 ? P.shard_mode : 0};
    if (std::memcmp(pkey, ctx->pix_key, sizeof(pkey)) != 0) {
        const int tiles_x = (W + ts - 1) / ts, tiles_y = (H + ts - 1) / ts;
        std::vector<uint32_t> pix;
        pix.reserve(static_cast<size_t>(W) * H);
        for (int y = 0; y < H; ++y)
            for (int x = 0; x < W; ++x)
                if (tile_mine(P, (y / ts) * tiles_x + x / ts, tiles_x * tiles_y))
                    pix.push_back(static_cast<uint32_t>(y * W + x));
        ctx->pix_mem.ensure(std::max<size_t>(pix.size(), 1) * 4);
        cuda_check(cudaMemcpyAsync(ctx->pix_mem.p, pix.data(), pix.size() * 4ull, cudaMemcpyHostToDevice,
                                   ctx->stream), "H2D pixels");
        cuda_check(cudaStreamSynchronize(ctx->stream), "H2D pixels");
        ctx->pix_n = static_cast<uint32_t>(pix.size());
        std::memcpy(ctx->pix_key, pkey, sizeof(pkey));
    }
    const uint32_t n_pix = ctx->pix_n;
    const uint32_t* d_pix_all = ctx->pix_mem.as<uint32_t>();

    // Pass lanes: with 2, consecutive passes alternate between two stream
    // pairs with their own path state, so one pass's latency-bound shading
    // overlaps the other's issue-bound traversal (MCG_LANES=1: one pass at a
    // time). Deterministic mode keeps one lane: its epochs are (pass, bounce).
    const char* lanes_env = std::getenv("MCG_LANES");
    int lanes = lanes_env ? std::max(1, std::min(mcg_ctx::kMaxLanes, std::atoi(lanes_env))) : kDefaultLanes;
    if (deferred) lanes = 1;
    uint32_t k = P.samples_per_pass > 0 ? static_cast<uint32_t>(P.samples_per_pass) : 0;
    if (k == 0) {
        // paths in flight per pass: ~4M with one lane (measured 1M 866 ms,
        // 2M 773, 4M 751, 8M 769 per bench render), ~2M per lane with two
        // (1080p, same call: one lane 6.2M 658 ms; two lanes 2.1M 657, 4.1M
        // 648); MCG_PASS_PATHS overrides (experiments)
        const char* pp_env = std::getenv("MCG_PASS_PATHS");
        const uint64_t target = pp_env ? std::max<uint64_t>(1, std::strtoull(pp_env, nullptr, 10))
                                       : (lanes > 1 ? (1u << 21) : (1u << 22));
        k = static_cast<uint32_t>(std::max<uint64_t>(1, (target + n_pix - 1) / std::max<uint32_t>(n_pix, 1)));
    }
    k = std::min<uint32_t>(std::min<uint32_t>(k, 32u), static_cast<uint32_t>(P.spp));
    const uint64_t wh = static_cast<uint64_t>(W) * H;
    if (deferred && (static_cast<uint64_t>(k) * wh) >= (1ull << 26)) {
        fail(MCG_ERR_INVALID_ARGUMENT, "deterministic mode: samples_per_pass * pixels must be < 2^26");
    }
    const uint64_t max_paths = static_cast<uint64_t>(n_pix) * k;

    // Cache: external table, or the context's own one (tracer.hpp:67-68).
    mcg_cache* cache = nullptr;
    if (cache_on) {
        cache = external;
        if (!cache) {
            if (!ctx->own_cache || ctx->own_cache->n_cells != P.n_cells ||
                ctx->own_cache->n_entries != P.n_entries) {
                if (ctx->own_cache) mcg_cache_destroy(ctx->own_cache);
                ctx->own_cache = nullptr;
                const mcg_status s = mcg_cache_create(ctx, P.n_cells, P.n_entries, &ctx->own_cache);
                if (s != MCG_OK) fail(s, mcg_last_error());
            } else {
                const mcg_status s = mcg_cache_clear(ctx->own_cache);
                if (s != MCG_OK) fail(s, mcg_last_error());
            }
            cache = ctx->own_cache;
        }
    }

    // Path state: 2 layouts x (4 float4 + pid) + the hit record (float4) +
    // 1 float4 final radiance per path; shadow rays: 3 float4 + 1 byte per
    // (path, light); sort keys/values and the shadow queue as u32.
    const uint32_t n_lights = D.view.n_plights + D.view.n_rlights;
    const uint64_t n_shadow = max_paths * std::max<uint32_t>(1, n_lights);
    const size_t f4 = max_paths * sizeof(float4);
    if (static_cast<uint32_t>(P.spp) <= k) lanes = 1;   // a single pass
    const size_t lane_bytes = f4 * (2 * sizeof(PathRay) / 16 + 2 * sizeof(PathVal) / 16 + 1) + n_shadow * (48 + 4 + 1) + max_paths * 4 * 6 + n_pix * 4ull + 1024;
    ctx->path_mem.ensure(lane_bytes);
    for (int l = 1; l < lanes; ++l) ctx->lane_path[l].ensure(lane_bytes);
    RenderView R{};
    R.S = D.view;
    if (cache && cache->world > 1 && !cache->stripes) fail(MCG_ERR_INVALID_ARGUMENT, "striped table: attach the stripes first");
    R.C = cache ? cache->view() : mcgd::CacheView{nullptr, nullptr, 1, ~0ull, 1, 1, 1, nullptr, nullptr, nullptr, 0};
    // (a descriptor trace records lookups in the VM's order: no look-ahead
    // then; the where-hint packs into 8 bits)
    const bool look_ahead = look_ahead_req && R.C.trace == nullptr && R.C.n_entries < 255u;
    // MCG_LOOKAHEAD=2: the probe as its own kernel after each trace (else
    // fused into the trace kernels' hit-record epilogue)
    R.ahead_fused = look_ahead && !(la_env && std::string(la_env) == "2") ? 1u : 0u;
    R.cache_on = cache_on ? 1 : 0;
    R.mip_offset = P.mip_offset;
    camera_setup(D.cam, W, H, R.cam);
    std::memcpy(R.cam_pos, D.cam.cam_position, sizeof(R.cam_pos));
    R.W = W;
    R.H = H;
    R.max_bounces = P.max_bounces;
    R.seed = P.rng_seed;
    R.diffuse_spread = P.diffuse_spread;
    R.n_pix = n_pix;
    auto layout = [&](RenderView& V, char* base) {
        V.pa = reinterpret_cast<PathRay*>(base);          // 128 B per path
        V.pa2 = V.pa + max_paths;
        V.pb = reinterpret_cast<PathVal*>(V.pa2 + max_paths);   // 32 B
        V.pb2 = V.pb + max_paths;
        V.fin = reinterpret_cast<float4*>(V.pb2 + max_paths);   // 16 B
        V.ahead_on = look_ahead ? 1u : 0u;
        V.sro = V.fin + max_paths;
        V.srd = V.sro + n_shadow;
        V.scon = V.srd + n_shadow;
        uint32_t* u32 = reinterpret_cast<uint32_t*>(V.scon + n_shadow);
        V.keys = u32;
        V.vals = u32 + max_paths;
        uint32_t* skey_ = u32 + 2 * max_paths;
        uint32_t* order_ = u32 + 3 * max_paths;
        V.skey = skey_;
        V.order = order_;
        V.squeue = u32 + 6 * max_paths;
        V.pix = d_pix_all;
        V.shadow_count = reinterpret_cast<unsigned int*>(V.squeue + n_shadow + n_pix);
        V.vis = reinterpret_cast<uint8_t*>(V.shadow_count + 64);
    };
    R.radiance = d_rad;
    R.nodes_found = d_nodes;
    R.samples = d_samples;
    ctx->stats_mem.ensure(4096 + static_cast<size_t>(P.spp) * 8);
    R.stats = ctx->stats_mem.as<unsigned long long>();
    R.hps = R.stats + kStatCount;
    cuda_check(cudaMemsetAsync(R.stats, 0, (kStatCount + P.spp) * 8ull, ctx->stream), "memset stats");
    unsigned long long* cache_ctr = cache ? cache->counters : nullptr;

    if (deferred) {
        const uint64_t cap = max_paths * std::max<uint32_t>(1, D.max_cache_points);
        if (cap >= (1ull << 32)) fail(MCG_ERR_INVALID_ARGUMENT, "store queue too large");
        ctx->queue_mem.ensure(cap * 32 + 64);
        R.q.keys = ctx->queue_mem.as<unsigned long long>();
        R.q.vals = R.q.keys + cap;
        R.q.count = reinterpret_cast<unsigned int*>(R.q.keys + 4 * cap);
        R.q.capacity = static_cast<unsigned>(cap);
    }
    // Sort key (MCG_SORT): "dir3" (default) = slot | octant of the vertex's
    // bounce direction | Morton code of the hit point on a 2^6 grid (23 bits
    // with <= 4 slots: 3 radix passes); "morton" = slot | Morton 2^7;
    // "dir" = slot | normal octant + azimuth quadrant | Morton 2^6;
    // "material" = slot only. Measured per bench render (profiles/README.md):
    // dir3 716 ms, morton 741, dir 733, material 1383 (older build).
    const char* sort_env = std::getenv("MCG_SORT");
    const std::string sort_mode = sort_env ? std::string(sort_env) : std::string("dir3");
    const bool morton = sort_mode != "material";
    const int slot_bits = std::max(1, bits_for(D.view.n_programs));
    const char* mb_env = std::getenv("MCG_MORTON_BITS");   // 2^b cells per axis
    int mb = mb_env ? std::min(8, std::max(1, std::atoi(mb_env))) : (sort_mode == "morton" ? 7 : 6);
    if (!mb_env && sort_mode == "dir3") {
        // keep the key within 24 bits (three radix passes): scenes with more
        // materials and look-ahead bits give up Morton precision first
        const int pb = look_ahead ? static_cast<int>(std::min<uint32_t>(2u, D.max_cache_points)) : 0;
        while (mb > 4 && 3 * mb + 3 + pb + slot_bits > 24) --mb;
    }
    R.key_shift = (morton && slot_bits <= 8) ? static_cast<uint32_t>(3 * mb) : 0u;
    R.key_dir = 0u;
    if (R.key_shift && sort_mode == "dir") {
        R.key_dir = 1u;
        R.key_shift = 24u;  // the direction-class key keeps its 24-bit layout
    } else if (R.key_shift && sort_mode == "dir3") {
        R.key_dir = 2u;
        R.key_shift = static_cast<uint32_t>(3 * mb + 3);
    }
    for (int a = 0; a < 3; ++a) {
        const float ext = D.root_hi[a] - D.root_lo[a];
        R.box_lo[a] = D.root_lo[a];
        R.box_scale[a] = ext > 0.0f ? (static_cast<float>(1 << mb) - 0.001f) / ext : 0.0f;
    }
    // Look-ahead probes (MCG_LOOKAHEAD=0: off): the hit bits of the first
    // cache points (up to 2 key bits) go between the slot and the Morton part.
    R.key_pat = R.key_shift;
    R.pat_mask = 0u;
    if (look_ahead && R.key_shift) {
        const uint32_t pb = std::min<uint32_t>(2u, std::min(mcgd::kAhead, D.max_cache_points));
        R.pat_mask = (1u << pb) - 1u;
        R.key_shift += pb;
    }
    const int key_bits = static_cast<int>(R.key_shift) + slot_bits;
    // Shadow rays over the SAH tree of the reference's leaves (exact for
    // any-hit); MCG_SHADOW_TREE=ref keeps the reference's own tree.
    const char* stree_env = std::getenv("MCG_SHADOW_TREE");
    const bool sah_shadow = !(stree_env && std::string(stree_env) == "ref");
    // MCG_OVERLAP=0: shadow rays on the main stream (no concurrency)
    const char* ov_env = std::getenv("MCG_OVERLAP");
    const bool overlap = !(ov_env && std::string(ov_env) == "0");
    if (overlap && !ctx->aux) {
        cuda_check(cudaStreamCreateWithFlags(&ctx->aux, cudaStreamNonBlocking), "aux stream");
        cuda_check(cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming), "event");
        cuda_check(cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming), "event");
    }
    if (lanes > 1 && !ctx->ev_lane[0]) {
        for (cudaEvent_t& e : ctx->ev_lane) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    }
    for (int l = 1; l < lanes; ++l) {
        if (ctx->lane_stream[l]) continue;
        cuda_check(cudaStreamCreateWithFlags(&ctx->lane_stream[l], cudaStreamNonBlocking), "lane stream");
        cuda_check(cudaStreamCreateWithFlags(&ctx->lane_aux[l], cudaStreamNonBlocking), "aux stream");
        cuda_check(cudaEventCreateWithFlags(&ctx->lane_fork[l], cudaEventDisableTiming), "event");
        cuda_check(cudaEventCreateWithFlags(&ctx->lane_join[l], cudaEventDisableTiming), "event");
    }
    constexpr int kML = mcg_ctx::kMaxLanes;
    RenderView RL[kML];
    cudaStream_t lane_main[kML], lane_aux[kML];
    cudaEvent_t lane_fork[kML], lane_join[kML];
    mcg::DevMem* lane_tmp[kML];
    for (int l = 0; l < lanes; ++l) {
        RL[l] = R;
        layout(RL[l], (l == 0 ? ctx->path_mem : ctx->lane_path[l]).as<char>());
        lane_main[l] = l == 0 ? ctx->stream : ctx->lane_stream[l];
        lane_aux[l] = l == 0 ? ctx->aux : ctx->lane_aux[l];
        lane_fork[l] = l == 0 ? ctx->ev_fork : ctx->lane_fork[l];
        lane_join[l] = l == 0 ? ctx->ev_join : ctx->lane_join[l];
        lane_tmp[l] = l == 0 ? &ctx->cub_temp : &ctx->lane_cub[l];
    }
    const int block = MCG_SHADE_BLOCK;
    const int max_stack = static_cast<int>(D.max_stack);
    const size_t smem = static_cast<size_t>(max_stack) * block * 3 * sizeof(float);
    if (smem > 200 * 1024) fail(MCG_ERR_INVALID_ARGUMENT, "material stack too deep for shared memory");
#ifndef MCG_TRACE_CARVEOUT
#define MCG_TRACE_CARVEOUT 0
#endif
    // traversal kernels use no shared memory: ask for the whole L1 (the tree
    // and triangles are ~1 MB; 12% of the node loads miss L1). Same call:
    // 646.6 / 647.1 vs 649.2 / 648.5 ms per bench render.
    cudaFuncSetAttribute(k_trace_closest_ww<3>, cudaFuncAttributePreferredSharedMemoryCarveout, MCG_TRACE_CARVEOUT);
    cudaFuncSetAttribute(k_trace_closest_ww<mcgd::kAhead>, cudaFuncAttributePreferredSharedMemoryCarveout, MCG_TRACE_CARVEOUT);
    cudaFuncSetAttribute(k_shadow_ww<true>, cudaFuncAttributePreferredSharedMemoryCarveout, MCG_TRACE_CARVEOUT);
    cudaFuncSetAttribute(k_primary<3>, cudaFuncAttributePreferredSharedMemoryCarveout, MCG_TRACE_CARVEOUT);
    cudaFuncSetAttribute(k_primary<mcgd::kAhead>, cudaFuncAttributePreferredSharedMemoryCarveout, MCG_TRACE_CARVEOUT);
    // scenes whose materials have at most three cache points take the
    // kernels with the short, unrolled look-ahead loop
    const bool many_cps = D.max_cache_points > 3;
    // programs up to 32 KB of bytecode are staged in shared memory per block
    // (MCG_CODE_SMEM=0: read from global memory through L1)
    const char* cs_env = std::getenv("MCG_CODE_SMEM");
    const size_t code_bytes = static_cast<size_t>(D.view.n_code) * sizeof(mcg_insn);
    const bool code_smem = !(cs_env && std::string(cs_env) == "0") && code_bytes <= 32 * 1024;
    const size_t smem_launch = smem + (code_smem ? code_bytes : 0);
    cudaFuncSetAttribute(k_shade<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    cudaFuncSetAttribute(k_shade<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    cudaFuncSetAttribute(k_shade<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_launch));
    cudaFuncSetAttribute(k_shade<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_launch));
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    cuda_check(cudaEventCreate(&ev0), "event");
    cuda_check(cudaEventCreate(&ev1), "event");
    cuda_check(cudaEventRecord(ev0, ctx->stream), "event record");
    if (lanes > 1) {
        // the other lanes start after the setup (stats reset, pixel lists) on the main stream
        cuda_check(cudaEventRecord(ctx->ev_lane[kML], ctx->stream), "event record");
        for (int l = 1; l < lanes; ++l) cuda_check(cudaStreamWaitEvent(lane_main[l], ctx->ev_lane[kML], 0), "wait");
    }

    int prev_lane = -1;
    uint32_t pass = 0;
    for (uint32_t start = 0; start < static_cast<uint32_t>(P.spp); start += k, ++pass) {
        const int l = static_cast<int>(pass % static_cast<uint32_t>(lanes));
        const cudaStream_t sm = lane_main[l], sa = lane_aux[l];
        RenderView R = RL[l];   // the pass starts on the lane's first layout
        const uint32_t kk = std::min<uint32_t>(k, static_cast<uint32_t>(P.spp) - start);
        R.n_paths = n_pix * kk;
        R.sample0 = P.first_sample + start;
        R.hps_base = start;
        const unsigned grid = grid_for(R.n_paths, 256);
        {
            LaunchScope ls(ctx, "primary", 0.0, sm);
            if (many_cps) k_primary<mcgd::kAhead><<<grid_for(R.n_paths, MCG_PRIMARY_BLOCK), MCG_PRIMARY_BLOCK, 0, sm>>>(R);
            else k_primary<3><<<grid_for(R.n_paths, MCG_PRIMARY_BLOCK), MCG_PRIMARY_BLOCK, 0, sm>>>(R);
            ls.done();
        }
        if (look_ahead && !R.ahead_fused) {
            LaunchScope ls(ctx, "lookahead", 0.0, sm);
            k_lookahead<<<grid, 256, 0, sm>>>(R, nullptr);
            ls.done();
        }
        for (int b = 0; b <= P.max_bounces; ++b) {
            // Stable radix sort of (key -> layout position): hits in
            // material order first, paths without a hit (key n_programs) last.
            sort_pairs_u32(ctx, R.keys, const_cast<uint32_t*>(R.skey), R.vals, const_cast<uint32_t*>(R.order), R.n_paths,
                           key_bits, sm, lane_tmp[l]);
            // counters: [0] shadow rays queued, [1] shadow cursor, [2] live paths, [3] trace cursor
            cuda_check(cudaMemsetAsync(R.shadow_count, 0, 16, sm), "memset");
            if (deferred) cuda_check(cudaMemsetAsync(R.q.count, 0, 4, sm), "memset");
            {
                LaunchScope ls(ctx, "shade", 0.0, sm);
                const unsigned sg = grid_for(R.n_paths, block);
                R.shade_perm = scatter && !deferred ? coprime_near(sg, 0.6180339887) : 1u;
                const uint32_t wh32 = static_cast<uint32_t>(wh);
                // deterministic mode: stores are queued and applied after the
                // shade (NEE and the bounce need none of them)
                if (code_smem) {
                    if (deferred) k_shade<true, true><<<sg, block, smem_launch, sm>>>(R, R.skey, R.order, max_stack, wh32, b);
                    else k_shade<false, true><<<sg, block, smem_launch, sm>>>(R, R.skey, R.order, max_stack, wh32, b);
                } else {
                    if (deferred) k_shade<true, false><<<sg, block, smem, sm>>>(R, R.skey, R.order, max_stack, wh32, b);
                    else k_shade<false, false><<<sg, block, smem, sm>>>(R, R.skey, R.order, max_stack, wh32, b);
                }
                ls.done();
            }
            // the path state now lives at the sorted positions
            std::swap(R.pa, R.pa2);
            std::swap(R.pb, R.pb2);
            if (deferred) {   // one lane: sm == ctx->stream
                unsigned int count = 0;
                cuda_check(cudaMemcpyAsync(&count, R.q.count, 4, cudaMemcpyDeviceToHost, sm), "D2H");
                cuda_check(cudaStreamSynchronize(sm), "sync");
                if (count > R.q.capacity) fail(MCG_ERR_CUDA, "store queue overflow");
                if (count) {
                    const uint64_t cap = R.q.capacity;
                    unsigned long long* k1 = R.q.keys + 2 * cap;
                    unsigned long long* v1 = R.q.keys + 3 * cap;
                    sort_pairs_u64(ctx, R.q.keys, k1, R.q.vals, v1, count, 64);
                    // apply_ordered adds won/full at counters[2]/[3] == kStatWon/kStatFull.
                    apply_ordered(ctx, cache, k1, v1, count, 32, nullptr, nullptr, nullptr, R.stats);
                }
            }
            // Shadow rays (aux stream) and continuation rays (main stream)
            // of vertex b are independent; k_resolve_lights waits for both.
            const bool fork = overlap && n_lights && b < P.max_bounces;
            if (fork) {
                cuda_check(cudaEventRecord(lane_fork[l], sm), "event");
                cuda_check(cudaStreamWaitEvent(sa, lane_fork[l], 0), "wait");
            }
            if (n_lights) {
                cudaStream_t st = fork ? sa : sm;
                LaunchScope ls(ctx, "trace_shadow", 0.0, st);
                if (sah_shadow) k_shadow_ww<true><<<grid_for(n_shadow, MCG_SHADOW_BLOCK), MCG_SHADOW_BLOCK, 0, st>>>(R);
                else k_shadow_ww<false><<<grid_for(n_shadow, MCG_SHADOW_BLOCK), MCG_SHADOW_BLOCK, 0, st>>>(R);
                ls.done();
            }
            if (fork) cuda_check(cudaEventRecord(lane_join[l], sa), "event");
            if (b < P.max_bounces) {
                LaunchScope ls(ctx, "trace_closest", 0.0, sm);
                if (many_cps) {
                    k_trace_closest_ww<mcgd::kAhead><<<grid_for(R.n_paths, MCG_TRACE_BLOCK), MCG_TRACE_BLOCK, 0, sm>>>(
                        R, R.shadow_count + 2, b + 1);
                } else {
                    k_trace_closest_ww<3><<<grid_for(R.n_paths, MCG_TRACE_BLOCK), MCG_TRACE_BLOCK, 0, sm>>>(
                        R, R.shadow_count + 2, b + 1);
                }
                ls.done();
            }
            if (b < P.max_bounces && look_ahead && !R.ahead_fused) {
                LaunchScope ls(ctx, "lookahead", 0.0, sm);
                k_lookahead<<<grid, 256, 0, sm>>>(R, R.shadow_count + 2);
                ls.done();
            }
            if (fork) cuda_check(cudaStreamWaitEvent(sm, lane_join[l], 0), "wait");
            {
                LaunchScope ls(ctx, "resolve_lights", 0.0, sm);
                k_resolve_lights<<<grid, 256, 0, sm>>>(R, b);
                ls.done();
            }
        }
        // passes reach the framebuffers in sample order (the double
        // accumulators' summation order): wait for the previous pass's
        // accumulate when it ran on the other lane
        if (prev_lane >= 0 && prev_lane != l) cuda_check(cudaStreamWaitEvent(sm, ctx->ev_lane[prev_lane], 0), "wait");
        {
            LaunchScope ls(ctx, "accumulate", n_pix * (40.0 + 40.0 * kk), sm);
            k_accumulate<<<grid_for(n_pix, 256), 256, 0, sm>>>(R, kk);
            ls.done();
        }
        if (lanes > 1) cuda_check(cudaEventRecord(ctx->ev_lane[l], sm), "event record");
        prev_lane = l;
    }
    for (int l = 1; l < lanes; ++l) {   // the render ends when every lane is done
        cuda_check(cudaEventRecord(ctx->ev_lane[l], lane_main[l]), "event record");
        cuda_check(cudaStreamWaitEvent(ctx->stream, ctx->ev_lane[l], 0), "wait");
    }
    cuda_check(cudaEventRecord(ev1, ctx->stream), "event record");
    if (cache_ctr) {
        // Mirror the render's lookups/hits/inserts into the table's counters
        // (MaterialCache::counters after a render, cache.cpp:146-150), on the
        // render's stream (no host round trip, no legacy-stream sync).
        k_add_counters<<<1, 32, 0, ctx->stream>>>(cache_ctr, R.stats);
        ++ctx->launches;
    }
    unsigned long long st[kStatCount];
    cuda_check(cudaMemcpyAsync(st, R.stats, sizeof(st), cudaMemcpyDeviceToHost, ctx->stream), "D2H stats");
    if (stats && stats->hits_per_sample) {
        cuda_check(cudaMemcpyAsync(stats->hits_per_sample, R.hps, P.spp * 8ull, cudaMemcpyDeviceToHost, ctx->stream), "D2H hps");
    }
    cuda_check(cudaStreamSynchronize(ctx->stream), "render");
    float dev_ms = 0.0f;
    cudaEventElapsedTime(&dev_ms, ev0, ev1);
    cudaEventDestroy(ev0);
    cudaEventDestroy(ev1);
    const auto t1 = std::chrono::steady_clock::now();
    if (stats) {
        uint64_t* hps = stats->hits_per_sample;
        std::memset(stats, 0, sizeof(*stats));
        stats->hits_per_sample = hps;
        stats->wall_time_s = std::chrono::duration<double>(t1 - t0).count();
        stats->device_ms = dev_ms;
        stats->lookups = st[kStatLookups];
        stats->hits = st[kStatHits];
        stats->inserts_won = st[kStatWon];
        stats->inserts_lost_full = st[kStatFull];
        stats->stores_attempted = st[kStatStores];
        stats->stores_won = st[kStatWon];
        stats->instructions_executed = st[kStatInstrs];
        stats->max_stack_seen = D.max_stack;
        stats->paths = static_cast<uint64_t>(n_pix) * P.spp;
        stats->shading_points = st[kStatShade];
        stats->shadow_rays = st[kStatShadow];
        stats->bvh_nodes = st[kStatNodes] + st[kStatNodesShadow];
        stats->prims_tested = st[kStatPrims] + st[kStatPrimsShadow];
        stats->tex_samples = st[kStatTex];
        stats->bvh_nodes_shadow = st[kStatNodesShadow];
        stats->prims_tested_shadow = st[kStatPrimsShadow];
        stats->closest_rays = st[kStatClosestRays];
        stats->shadow_occluded = st[kStatOccluded];
        stats->launches = ctx->launches - launches0;
    }
}

// ---------------------------------------------------------------------------
// In-process multi-GPU render (mcg_options.n_devices > 1)
// ---------------------------------------------------------------------------

// NCCL, loaded at run time (the process may already hold torch's copy of
// libnccl.so.2; dlopen then returns that one): the five calls the frame
// gather needs, types from the system nccl.h.
struct NcclApi {
    bool loaded = false;
    std::string error;
    ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*group_start)() = nullptr;
    ncclResult_t (*group_end)() = nullptr;
    ncclResult_t (*reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t,
                           cudaStream_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            a.error = std::string("cannot load libnccl.so.2: ") + dlerror();
            return a;
        }
        a.comm_init_all = reinterpret_cast<decltype(a.comm_init_all)>(dlsym(h, "ncclCommInitAll"));
        a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        a.group_start = reinterpret_cast<decltype(a.group_start)>(dlsym(h, "ncclGroupStart"));
        a.group_end = reinterpret_cast<decltype(a.group_end)>(dlsym(h, "ncclGroupEnd"));
        a.reduce = reinterpret_cast<decltype(a.reduce)>(dlsym(h, "ncclReduce"));
        a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
        a.loaded = a.comm_init_all && a.comm_destroy && a.group_start && a.group_end && a.reduce && a.error_string;
        if (!a.loaded) a.error = "libnccl.so.2 lacks a required symbol";
        return a;
    }();
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) fail(MCG_ERR_CUDA, std::string(what) + ": " + nccl().error_string(r));
}

// Zeroes the frame outside this device's tiles, so the frames sum exactly.
__global__ void k_zero_unowned(double* rad, double* nodes, uint32_t* samples, int W, int H, int ts, int rank,
                               int count, int mode) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= static_cast<uint32_t>(W) * static_cast<uint32_t>(H)) return;
    const int x = static_cast<int>(i % static_cast<uint32_t>(W)), y = static_cast<int>(i / static_cast<uint32_t>(W));
    const int tiles_x = (W + ts - 1) / ts, n_tiles = tiles_x * ((H + ts - 1) / ts);
    const int tile = (y / ts) * tiles_x + x / ts;
    bool mine;
    if (mode == MCG_SHARD_INTERLEAVED) {
        mine = tile % count == rank;
    } else {
        const int lo = static_cast<int>(static_cast<int64_t>(n_tiles) * rank / count);
        const int hi = static_cast<int>(static_cast<int64_t>(n_tiles) * (rank + 1) / count);
        mine = tile >= lo && tile < hi;
    }
    if (mine) return;
    rad[3ull * i] = 0.0;
    rad[3ull * i + 1] = 0.0;
    rad[3ull * i + 2] = 0.0;
    nodes[i] = 0.0;
    samples[i] = 0u;
}

__global__ void k_add_frames(double* rad, double* nodes, uint32_t* samples, const double* rad2,
                             const double* nodes2, const uint32_t* samples2, size_t np) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i >= np) return;
    rad[3 * i] += rad2[3 * i];
    rad[3 * i + 1] += rad2[3 * i + 1];
    rad[3 * i + 2] += rad2[3 * i + 2];
    nodes[i] += nodes2[i];
    samples[i] += samples2[i];
}

void multi_render(mcg_ctx* ctx, const mcg_render_params& P, mcg_frame* frame, mcg_render_stats* stats) {
    const int n = 1 + static_cast<int>(ctx->peers.size());
    if (P.shard_count > 1) fail(MCG_ERR_INVALID_ARGUMENT, "a multi-device context shards the image itself");
    const int W = P.width ? P.width : ctx->scene.cam.cam_width;
    const int H = P.height ? P.height : ctx->scene.cam.cam_height;
    if (W <= 0 || H <= 0) fail(MCG_ERR_INVALID_ARGUMENT, "image size must be positive");
    const auto t0 = std::chrono::steady_clock::now();
    const size_t np = static_cast<size_t>(W) * H;
    std::vector<mcg_ctx*> all{ctx};
    all.insert(all.end(), ctx->peers.begin(), ctx->peers.end());
    std::vector<mcg_render_stats> st(n);
    std::vector<std::vector<uint64_t>> hps(n, std::vector<uint64_t>(static_cast<size_t>(std::max(P.spp, 0)), 0));
    std::vector<std::exception_ptr> err(n);
    std::vector<std::string> msg(n);
    std::vector<mcg_status> code(n, MCG_OK);
    // one host thread per device: render its tiles into a device frame that
    // starts as the caller's frame, then zero everything outside its tiles
    auto work = [&](int r) {
        mcg_ctx* c = all[r];
        try {
            cuda_check(cudaSetDevice(c->device), "cudaSetDevice");
            c->scratch_e.ensure(np * 44 + 64);
            double* rad = c->scratch_e.as<double>();
            double* nodes = rad + 3 * np;
            uint32_t* samples = reinterpret_cast<uint32_t*>(nodes + np);
            cuda_check(cudaMemcpyAsync(rad, frame->radiance, np * 24, cudaMemcpyHostToDevice, c->stream), "H2D frame");
            cuda_check(cudaMemcpyAsync(nodes, frame->nodes_found, np * 8, cudaMemcpyHostToDevice, c->stream), "H2D frame");
            cuda_check(cudaMemcpyAsync(samples, frame->samples, np * 4, cudaMemcpyHostToDevice, c->stream), "H2D frame");
            mcg_render_params pr = P;
            pr.shard_rank = r;
            pr.shard_count = n;
            st[r].hits_per_sample = hps[r].data();
            render_device(c, pr, nullptr, rad, nodes, samples, &st[r]);
            const int ts = P.tile_size > 0 ? P.tile_size : 16;
            k_zero_unowned<<<grid_for(np, 256), 256, 0, c->stream>>>(rad, nodes, samples, W, H, ts, r, n, P.shard_mode);
            cuda_check(cudaGetLastError(), "k_zero_unowned");
            ++c->launches;
            cuda_check(cudaStreamSynchronize(c->stream), "render");
        } catch (const mcg::Failure& e) {
            code[r] = e.code;
            msg[r] = e.what();
        } catch (...) {
            err[r] = std::current_exception();
        }
    };
    std::vector<std::thread> threads;
    for (int r = 1; r < n; ++r) threads.emplace_back(work, r);
    work(0);
    for (auto& t : threads) t.join();
    for (int r = 0; r < n; ++r) {
        if (err[r]) std::rethrow_exception(err[r]);
        if (code[r] != MCG_OK) fail(code[r], "device " + std::to_string(all[r]->device) + ": " + msg[r]);
    }
    auto frame_of = [&](mcg_ctx* c, double*& rad, double*& nodes, uint32_t*& samples) {
        rad = c->scratch_e.as<double>();
        nodes = rad + 3 * np;
        samples = reinterpret_cast<uint32_t*>(nodes + np);
    };
    double *rad0, *nodes0;
    uint32_t* samples0;
    frame_of(ctx, rad0, nodes0, samples0);
    if (ctx->devices_distinct) {
        // the framebuffer gather over NVLink: ncclReduce(sum) to the first
        // device, one group over the three buffers of every device
        const NcclApi& api = nccl();
        if (!api.loaded) fail(MCG_ERR_CUDA, api.error);
        if (ctx->nccl_comms.size() != static_cast<size_t>(n)) {
            std::vector<int> devs(n);
            for (int r = 0; r < n; ++r) devs[r] = all[r]->device;
            std::vector<ncclComm_t> comms(n);
            nccl_check(api.comm_init_all(comms.data(), n, devs.data()), "ncclCommInitAll");
            ctx->nccl_comms.assign(comms.begin(), comms.end());
        }
        nccl_check(api.group_start(), "ncclGroupStart");
        for (int r = 0; r < n; ++r) {
            double *rad, *nodes;
            uint32_t* samples;
            frame_of(all[r], rad, nodes, samples);
            ncclComm_t comm = static_cast<ncclComm_t>(ctx->nccl_comms[r]);
            nccl_check(api.reduce(rad, rad, 3 * np, ncclFloat64, ncclSum, 0, comm, all[r]->stream), "ncclReduce");
            nccl_check(api.reduce(nodes, nodes, np, ncclFloat64, ncclSum, 0, comm, all[r]->stream), "ncclReduce");
            nccl_check(api.reduce(samples, samples, np, ncclUint32, ncclSum, 0, comm, all[r]->stream), "ncclReduce");
        }
        nccl_check(api.group_end(), "ncclGroupEnd");
        for (int r = 1; r < n; ++r) {
            cuda_check(cudaSetDevice(all[r]->device), "cudaSetDevice");
            cuda_check(cudaStreamSynchronize(all[r]->stream), "ncclReduce");
        }
        cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
    } else {
        // a device listed twice (tests on one GPU): copy each frame to the
        // first device and add it there (same exact sum)
        cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
        ctx->gather_tmp.ensure(np * 44 + 64);
        double* rad2 = ctx->gather_tmp.as<double>();
        double* nodes2 = rad2 + 3 * np;
        uint32_t* samples2 = reinterpret_cast<uint32_t*>(nodes2 + np);
        for (int r = 1; r < n; ++r) {
            double *rad, *nodes;
            uint32_t* samples;
            frame_of(all[r], rad, nodes, samples);
            cuda_check(cudaMemcpyPeerAsync(rad2, ctx->device, rad, all[r]->device, np * 36, ctx->stream), "gather");
            k_add_frames<<<grid_for(np, 256), 256, 0, ctx->stream>>>(rad0, nodes0, samples0, rad2, nodes2, samples2, np);
            cuda_check(cudaGetLastError(), "k_add_frames");
            ++ctx->launches;
        }
    }
    cuda_check(cudaMemcpyAsync(frame->radiance, rad0, np * 24, cudaMemcpyDeviceToHost, ctx->stream), "D2H frame");
    cuda_check(cudaMemcpyAsync(frame->nodes_found, nodes0, np * 8, cudaMemcpyDeviceToHost, ctx->stream), "D2H frame");
    cuda_check(cudaMemcpyAsync(frame->samples, samples0, np * 4, cudaMemcpyDeviceToHost, ctx->stream), "D2H frame");
    cuda_check(cudaStreamSynchronize(ctx->stream), "render");
    if (stats) {
        uint64_t* out_hps = stats->hits_per_sample;
        mcg_render_stats sum = st[0];
        for (int r = 1; r < n; ++r) {
            const mcg_render_stats& x = st[r];
            sum.lookups += x.lookups;
            sum.hits += x.hits;
            sum.inserts_won += x.inserts_won;
            sum.inserts_lost_full += x.inserts_lost_full;
            sum.stores_attempted += x.stores_attempted;
            sum.stores_won += x.stores_won;
            sum.instructions_executed += x.instructions_executed;
            sum.paths += x.paths;
            sum.shading_points += x.shading_points;
            sum.shadow_rays += x.shadow_rays;
            sum.bvh_nodes += x.bvh_nodes;
            sum.prims_tested += x.prims_tested;
            sum.tex_samples += x.tex_samples;
            sum.bvh_nodes_shadow += x.bvh_nodes_shadow;
            sum.prims_tested_shadow += x.prims_tested_shadow;
            sum.closest_rays += x.closest_rays;
            sum.shadow_occluded += x.shadow_occluded;
            sum.launches += x.launches;
            sum.device_ms = std::max(sum.device_ms, x.device_ms);
        }
        sum.launches += static_cast<uint64_t>(n) + (ctx->devices_distinct ? 0u : static_cast<uint64_t>(n - 1));
        sum.wall_time_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        sum.hits_per_sample = out_hps;
        if (out_hps) {
            for (int sidx = 0; sidx < P.spp; ++sidx) {
                uint64_t a = 0;
                for (int r = 0; r < n; ++r) a += hps[r][sidx];
                out_hps[sidx] = a;
            }
        }
        *stats = sum;
    }
}

}  // namespace

namespace mcg {
void nccl_destroy(mcg_ctx* ctx) {
    if (ctx->nccl_comms.empty()) return;
    const NcclApi& api = nccl();
    if (api.loaded) {
        for (void* c : ctx->nccl_comms) api.comm_destroy(static_cast<ncclComm_t>(c));
    }
    ctx->nccl_comms.clear();
}
}  // namespace mcg

extern "C" {

mcg_status mcg_intersect_batch(mcg_ctx* ctx, const float* rays, size_t n, float t_min, float t_max,
                               int32_t variant, float* out) {
    return guarded([&] {
        if (!ctx || (n && (!rays || !out))) fail(MCG_ERR_INVALID_ARGUMENT, "null argument");
        if (!ctx->scene.loaded) fail(MCG_ERR_INVALID_ARGUMENT, "no scene uploaded");
        if (variant < 0 || variant > 4) fail(MCG_ERR_INVALID_ARGUMENT, "variant must be 0..4");
        if (n >= (1ull << 31)) fail(MCG_ERR_INVALID_ARGUMENT, "batch too large");
        if (!n) return;
        ctx->scratch_a.ensure(n * 24);
        ctx->scratch_b.ensure(n * 96);
        float* dr = ctx->scratch_a.as<float>();
        float* dout = ctx->scratch_b.as<float>();
        cuda_check(cudaMemcpyAsync(dr, rays, n * 24, cudaMemcpyHostToDevice, ctx->stream), "H2D rays");
        const mcgd::SceneView& S = ctx->scene.view;
        const uint32_t n32 = static_cast<uint32_t>(n);
        const unsigned g = grid_for(n, 256);
        {
            const int depth = static_cast<int>(ctx->scene.max_stack4) + 1;
            const size_t pk_bytes = 8ull * depth * (2 + 32) * sizeof(float);
            if (variant == 4) pk_smem_attr(pk_bytes);
            LaunchScope ls(ctx, "intersect_batch", 0.0);
            if (variant == 0) k_intersect_batch<0><<<g, 256, 0, ctx->stream>>>(S, dr, n32, t_min, t_max, dout, 0);
            else if (variant == 1) k_intersect_batch<1><<<g, 256, 0, ctx->stream>>>(S, dr, n32, t_min, t_max, dout, 0);
            else if (variant == 2) k_intersect_batch<2><<<g, 256, 0, ctx->stream>>>(S, dr, n32, t_min, t_max, dout, 0);
            else if (variant == 3) k_intersect_batch<3><<<g, 256, 0, ctx->stream>>>(S, dr, n32, t_min, t_max, dout, 0);
            else k_intersect_batch<4><<<g, 256, pk_bytes, ctx->stream>>>(S, dr, n32, t_min, t_max, dout, depth);
            ls.done();
        }
        cuda_check(cudaMemcpyAsync(out, dout, n * 96, cudaMemcpyDeviceToHost, ctx->stream), "D2H hits");
        cuda_check(cudaStreamSynchronize(ctx->stream), "intersect_batch");
    });
}

mcg_status mcg_occluded_batch(mcg_ctx* ctx, const float* rays, size_t n, float t_min, const float* t_max,
                              int32_t variant, uint8_t* out) {
    return guarded([&] {
        if (!ctx || (n && (!rays || !t_max || !out))) fail(MCG_ERR_INVALID_ARGUMENT, "null argument");
        if (!ctx->scene.loaded) fail(MCG_ERR_INVALID_ARGUMENT, "no scene uploaded");
        if (variant < 0 || variant > 5) fail(MCG_ERR_INVALID_ARGUMENT, "variant must be 0..5");
        if (n >= (1ull << 31)) fail(MCG_ERR_INVALID_ARGUMENT, "batch too large");
        if (!n) return;
        ctx->scratch_a.ensure(n * 24);
        ctx->scratch_b.ensure(n * 4);
        ctx->scratch_c.ensure(n);
        float* dr = ctx->scratch_a.as<float>();
        float* dt = ctx->scratch_b.as<float>();
        uint8_t* dout = ctx->scratch_c.as<uint8_t>();
        cuda_check(cudaMemcpyAsync(dr, rays, n * 24, cudaMemcpyHostToDevice, ctx->stream), "H2D rays");
        cuda_check(cudaMemcpyAsync(dt, t_max, n * 4, cudaMemcpyHostToDevice, ctx->stream), "H2D tmax");
        const mcgd::SceneView& S = ctx->scene.view;
        const uint32_t n32 = static_cast<uint32_t>(n);
        const unsigned g = grid_for(n, 256);
        {
            const int depth = static_cast<int>(ctx->scene.max_stack4) + 1;
            const size_t pk_bytes = 8ull * depth * 2 * sizeof(float);
            if (variant == 4) pk_smem_attr(pk_bytes);
            LaunchScope ls(ctx, "occluded_batch", 0.0);
            if (variant == 0) k_occluded_batch<0><<<g, 256, 0, ctx->stream>>>(S, dr, n32, t_min, dt, dout, 0);
            else if (variant == 1) k_occluded_batch<1><<<g, 256, 0, ctx->stream>>>(S, dr, n32, t_min, dt, dout, 0);
            else if (variant == 2) k_occluded_batch<2><<<g, 256, 0, ctx->stream>>>(S, dr, n32, t_min, dt, dout, 0);
            else if (variant == 3) k_occluded_batch<3><<<g, 256, 0, ctx->stream>>>(S, dr, n32, t_min, dt, dout, 0);
            else if (variant == 5) k_occluded_batch<5><<<g, 256, 0, ctx->stream>>>(S, dr, n32, t_min, dt, dout, 0);
            else k_occluded_batch<4><<<g, 256, pk_bytes, ctx->stream>>>(S, dr, n32, t_min, dt, dout, depth);
            ls.done();
        }
        cuda_check(cudaMemcpyAsync(out, dout, n, cudaMemcpyDeviceToHost, ctx->stream), "D2H occluded");
        cuda_check(cudaStreamSynchronize(ctx->stream), "occluded_batch");
    });
}

mcg_status mcg_render_device(mcg_ctx* ctx, const mcg_render_params* params, mcg_cache* cache,
                             mcg_frame* d_frame, mcg_render_stats* stats) {
    return guarded([&] {
        if (!ctx || !params || !d_frame) fail(MCG_ERR_INVALID_ARGUMENT, "null argument");
        if (!ctx->peers.empty()) fail(MCG_ERR_INVALID_ARGUMENT, "a multi-device context renders through mcg_render");
        cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
        render_device(ctx, *params, cache, d_frame->radiance, d_frame->nodes_found,
                      d_frame->samples, stats);
    });
}

mcg_status mcg_render(mcg_ctx* ctx, const mcg_render_params* params, mcg_cache* cache,
                      mcg_frame* frame, mcg_render_stats* stats) {
    return guarded([&] {
        if (!ctx || !params || !frame || !frame->radiance || !frame->nodes_found || !frame->samples) {
            fail(MCG_ERR_INVALID_ARGUMENT, "null argument");
        }
        if (!ctx->scene.loaded) fail(MCG_ERR_INVALID_ARGUMENT, "no scene uploaded");
        cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
        if (!ctx->peers.empty()) {
            if (cache) fail(MCG_ERR_INVALID_ARGUMENT, "a multi-device context keeps one cache replica per device "
                                                      "(no external cache)");
            multi_render(ctx, *params, frame, stats);
            return;
        }
        const int W = params->width ? params->width : ctx->scene.cam.cam_width;
        const int H = params->height ? params->height : ctx->scene.cam.cam_height;
        if (W <= 0 || H <= 0) fail(MCG_ERR_INVALID_ARGUMENT, "image size must be positive");
        const size_t np = static_cast<size_t>(W) * H;
        ctx->scratch_e.ensure(np * 44 + 64);
        double* rad = ctx->scratch_e.as<double>();
        double* nodes = rad + 3 * np;
        uint32_t* samples = reinterpret_cast<uint32_t*>(nodes + np);
        cuda_check(cudaMemcpyAsync(rad, frame->radiance, np * 24, cudaMemcpyHostToDevice, ctx->stream), "H2D frame");
        cuda_check(cudaMemcpyAsync(nodes, frame->nodes_found, np * 8, cudaMemcpyHostToDevice, ctx->stream), "H2D frame");
        cuda_check(cudaMemcpyAsync(samples, frame->samples, np * 4, cudaMemcpyHostToDevice, ctx->stream), "H2D frame");
        render_device(ctx, *params, cache, rad, nodes, samples, stats);
        cuda_check(cudaMemcpyAsync(frame->radiance, rad, np * 24, cudaMemcpyDeviceToHost, ctx->stream), "D2H frame");
        cuda_check(cudaMemcpyAsync(frame->nodes_found, nodes, np * 8, cudaMemcpyDeviceToHost, ctx->stream), "D2H frame");
        cuda_check(cudaMemcpyAsync(frame->samples, samples, np * 4, cudaMemcpyDeviceToHost, ctx->stream), "D2H frame");
        cuda_check(cudaStreamSynchronize(ctx->stream), "render");
    });
}

}  // extern "C"

// ref_harness.cpp — TEST INFRASTRUCTURE. Links the reference's own sources
// (compiled in place from /root/reference/proj/core/src by oracle/Makefile
// into oracle/_ref/libmcref.so) and exposes them through extern "C" entry
// points for ctypes. Nothing here is shipped or measured as the product; it
// is the checker the C oracle (oracle/mc_oracle.c) and the CUDA path are
// pinned against, and the "reference" CPU baseline of bench.py.
//
// The reference's render() has no body (tracer.hpp:69-70 declares it,
// src/tracer.cpp is absent). ref_render() below restates it per
// tracer.hpp:7-94 and SPEC.md:378-434 with the decisions pinned in
// DESIGN.md §render, calling the reference's own Scene::intersect/occluded,
// footprint_gradients, execute and MaterialCache for everything they cover.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <sstream>
#include <thread>
#include <vector>

#include "matcache/analysis.hpp"
#include "matcache/cache.hpp"
#include "matcache/eval.hpp"
#include "matcache/graph.hpp"
#include "matcache/image.hpp"
#include "matcache/noise.hpp"
#include "matcache/raycone.hpp"
#include "matcache/rng.hpp"
#include "matcache/scene.hpp"
#include "matcache/stackvm.hpp"
#include "matcache/texture.hpp"
#include "matcache/value.hpp"
#include "mc_detmath.h"

using namespace matcache;

// Access to private members without touching the reference (explicit
// template instantiation may name private members): Scene's BVH
// (scene.hpp:114-118), read for the node-for-node tree comparison, and
// MaterialCache's slot array and won-insert counter (cache.hpp:105-113),
// used by the deferred (deterministic-insert) render below to take back a
// shading point's immediate inserts and re-apply them at the epoch's end
// through MaterialCache::update itself.
namespace {
template <typename Tag, typename Tag::type M>
struct Expose {
    friend typename Tag::type member(Tag) { return M; }
};
struct BvhTag {
    using type = std::vector<detail::BvhNode> Scene::*;
    friend type member(BvhTag);
};
template struct Expose<BvhTag, &Scene::bvh_>;
struct TableTag {
    using type = std::unique_ptr<std::atomic<uint64_t>[]> MaterialCache::*;
    friend type member(TableTag);
};
template struct Expose<TableTag, &MaterialCache::table_>;
struct WonTag {
    using type = std::atomic<uint64_t> MaterialCache::*;
    friend type member(WonTag);
};
template struct Expose<WonTag, &MaterialCache::inserts_won_>;
}  // namespace

namespace {

thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
    try {
        g_err.clear();
        f();
        return 0;
    } catch (const GraphError& e) {
        g_err = e.what();
        return 3;
    } catch (const CompileError& e) {
        g_err = e.what();
        return 4;
    } catch (const SceneError& e) {
        g_err = e.what();
        return 5;
    } catch (const ImageIoError& e) {
        g_err = e.what();
        return 6;
    } catch (const std::overflow_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 7;
    }
}

Vec3 v3(const float* p) { return {p[0], p[1], p[2]}; }
Vec2 v2(const float* p) { return {p[0], p[1]}; }

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- descriptor pipeline --------------------------------------------------
void ref_hash(const CacheDescriptor* d, size_t n, uint64_t* cell, uint32_t* check) {
    for (size_t i = 0; i < n; ++i) {
        cell[i] = hash_cell(d[i]);
        check[i] = hash_check(d[i]);
    }
}
void ref_encode(const float* rgb, size_t n, uint32_t* out) {
    for (size_t i = 0; i < n; ++i) out[i] = encode_value({rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]});
}
void ref_decode(const uint32_t* in, size_t n, float* rgb) {
    for (size_t i = 0; i < n; ++i) {
        const Color3 c = decode_value(in[i]);
        rgb[3 * i] = c.r;
        rgb[3 * i + 1] = c.g;
        rgb[3 * i + 2] = c.b;
    }
}
void ref_mip_texel(const float* uv, const float* g1, const float* g2, size_t n, int off,
                   uint8_t* mip, uint32_t* txy) {
    for (size_t i = 0; i < n; ++i) {
        mip[i] = mip_level(v2(g1 + 2 * i), v2(g2 + 2 * i), off);
        const auto [x, y] = texel_indices(v2(uv + 2 * i), mip[i]);
        txy[2 * i] = x;
        txy[2 * i + 1] = y;
    }
}
// in: 17 floats per item (cone width, spread, incoming3, normal3, e1 3, e2 3, duv1 2, duv2 2)
// minus spread... layout: width, incoming[3], normal[3], e1[3], e2[3], duv1[2], duv2[2] = 17
void ref_footprint(const float* in, size_t n, float* out) {
    for (size_t i = 0; i < n; ++i) {
        const float* p = in + 17 * i;
        RayCone c{p[0], 0.0f};
        UvPatch patch{v3(p + 7), v3(p + 10), v2(p + 13), v2(p + 15)};
        const auto [g1, g2] = footprint_gradients(c, v3(p + 1), v3(p + 4), patch);
        out[4 * i] = g1.x;
        out[4 * i + 1] = g1.y;
        out[4 * i + 2] = g2.x;
        out[4 * i + 3] = g2.y;
    }
}
float ref_cone_spread(float vfov_radians, int height) {
    return cone_for_camera(vfov_radians, height).spread;
}
void ref_rng(uint64_t seed, const uint64_t* pixel, const uint64_t* sample, const uint32_t* dim,
             size_t n, float* out) {
    for (size_t i = 0; i < n; ++i) out[i] = PathRng(seed, pixel[i], sample[i]).sample(dim[i]);
}
void ref_fbm(const int32_t* octaves, const float* fp, const float* uv, size_t n, float* out) {
    for (size_t i = 0; i < n; ++i) {
        NoiseParams p;
        p.octaves = octaves[i];
        p.frequency = fp[3 * i];
        p.lacunarity = fp[3 * i + 1];
        p.gain = fp[3 * i + 2];
        out[i] = fbm2(p, v2(uv + 2 * i));
    }
}
void ref_perlin(const float* xy, size_t n, float* out) {
    for (size_t i = 0; i < n; ++i) out[i] = perlin2(xy[2 * i], xy[2 * i + 1]);
}
void ref_sin_wave(const float* x, size_t n, float* out) {
    for (size_t i = 0; i < n; ++i) out[i] = ops::sin_wave(Value::scalar(x[i])).as_scalar();
}
void ref_power(const float* x, const float* y, size_t n, float* out) {
    for (size_t i = 0; i < n; ++i) {
        out[i] = ops::power(Value::scalar(x[i]), Value::scalar(y[i])).as_scalar();
    }
}
void ref_checker(float scale, const float* uv, size_t n, float* out) {
    for (size_t i = 0; i < n; ++i) out[i] = checker(scale, v2(uv + 2 * i));
}
// image: w*h RGB floats
void ref_bilinear(const float* img, int w, int h, int clamp, const float* uv, size_t n,
                  float* out) {
    ImageF im(w, h);
    for (int i = 0; i < w * h; ++i) im.pixels[i] = {img[3 * i], img[3 * i + 1], img[3 * i + 2]};
    for (size_t i = 0; i < n; ++i) {
        const Color3 c = sample_bilinear(im, v2(uv + 2 * i), clamp ? WrapMode::Clamp : WrapMode::Repeat);
        out[3 * i] = c.r;
        out[3 * i + 1] = c.g;
        out[3 * i + 2] = c.b;
    }
}
int ref_memory_bytes(uint64_t nc, uint64_t ne, uint64_t* out) {
    return guard([&] { *out = memory_bytes(nc, ne); });
}

// ---- MaterialCache --------------------------------------------------------
int ref_cache_new(uint64_t nc, uint32_t ne, void** out) {
    return guard([&] { *out = new MaterialCache(nc, ne); });
}
void ref_cache_free(void* c) { delete static_cast<MaterialCache*>(c); }
void ref_cache_update(void* c, const CacheDescriptor* d, const float* rgb, size_t n,
                      uint8_t* outcome, uint64_t* slot, uint64_t* packed) {
    auto* cache = static_cast<MaterialCache*>(c);
    for (size_t i = 0; i < n; ++i) {
        const UpdateResult r = cache->update(d[i], {rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]});
        if (outcome) outcome[i] = static_cast<uint8_t>(r.outcome);
        if (slot) slot[i] = r.slot;
        if (packed) packed[i] = r.packed;
    }
}
void ref_cache_lookup(void* c, const CacheDescriptor* d, size_t n, uint8_t* hit, float* rgb) {
    auto* cache = static_cast<MaterialCache*>(c);
    for (size_t i = 0; i < n; ++i) {
        const auto r = cache->lookup(d[i]);
        hit[i] = r.has_value();
        const Color3 v = r.value_or(Color3{});
        rgb[3 * i] = v.r;
        rgb[3 * i + 1] = v.g;
        rgb[3 * i + 2] = v.b;
    }
}
// CPU leg of the probe microbenchmark: the reference's own
// MaterialCache::update (phase 0, insert-all) or ::lookup (phase 1) over n
// descriptors from the device benchmark's generator (one splitmix64 per
// descriptor: mat < 8, node < 256, mip <= 16, texels uniform in 2^mip),
// split into contiguous ranges over `threads` std::threads. Returns the wall
// seconds; the payload of an insert is a constant colour.
double ref_probe_bench(void* c, uint64_t n, uint64_t seed, int phase, int threads) {
    auto* cache = static_cast<MaterialCache*>(c);
    const int nt = threads > 0 ? threads : 1;
    auto work = [&](uint64_t lo, uint64_t hi) {
        uint64_t found = 0;
        for (uint64_t i = lo; i < hi; ++i) {
            const uint64_t h = mix64(seed + 0x9e3779b97f4a7c15ull * (i + 1));
            const uint32_t w0 = static_cast<uint32_t>(h), w1 = static_cast<uint32_t>(h >> 32);
            const uint32_t mip = (w0 >> 11) % 17u, mask = (1u << mip) - 1u;
            CacheDescriptor d;
            d.mat_idx = w0 & 7u;
            d.node_idx = (w0 >> 3) & 255u;
            d.mip_level = static_cast<uint8_t>(mip);
            d.texel_x = w1 & mask;
            d.texel_y = (w1 >> 16) & mask;
            if (phase == 0) {
                cache->update(d, Color3{0.25f, 0.5f, 0.75f});
            } else {
                found += cache->lookup(d).has_value();
            }
        }
        return found;
    };
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 0; t < nt; ++t) {
        const uint64_t lo = n * t / nt, hi = n * (t + 1) / nt;
        pool.emplace_back([&, lo, hi] { work(lo, hi); });
    }
    for (auto& th : pool) th.join();
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

void ref_cache_slots(void* c, uint64_t first, size_t n, uint64_t* out) {
    auto* cache = static_cast<MaterialCache*>(c);
    for (size_t i = 0; i < n; ++i) out[i] = cache->slot_word(first + i);
}
void ref_cache_counters(void* c, uint64_t out[5]) {
    auto* cache = static_cast<MaterialCache*>(c);
    const auto k = cache->counters();
    out[0] = k.lookups;
    out[1] = k.hits;
    out[2] = k.inserts_won;
    out[3] = k.inserts_lost_full;
    out[4] = cache->occupied_slots();
}
int ref_cache_dump(void* c, const char* path) {
    return guard([&] { static_cast<MaterialCache*>(c)->dump(path); });
}
int ref_audit(const char* path, uint64_t out[4], char* problem, size_t cap) {
    const AuditReport r = audit_dump(path);
    out[0] = r.n_cells;
    out[1] = r.n_entries;
    out[2] = r.occupied;
    out[3] = static_cast<uint64_t>(r.bad_cell);
    std::snprintf(problem, cap, "%s", r.problem.c_str());
    return r.clean ? 1 : 0;
}

// ---- scenes, compiled programs, execute -----------------------------------
int ref_scene_load(const char* path, int min_subtree, void** out) {
    return guard([&] {
        AnalysisOptions opt;
        opt.min_subtree_size = min_subtree;
        *out = new Scene(load_scene(path, opt));
    });
}
void ref_scene_free(void* s) { delete static_cast<Scene*>(s); }
int ref_scene_materials(void* s) { return static_cast<int>(static_cast<Scene*>(s)->materials.size()); }

static void copy_text(const std::string& t, char* buf, size_t cap, size_t* len) {
    *len = t.size();
    if (buf && cap) {
        const size_t n = std::min(cap - 1, t.size());
        std::memcpy(buf, t.data(), n);
        buf[n] = 0;
    }
}
void ref_scene_disassemble(void* s, int slot, char* buf, size_t cap, size_t* len) {
    copy_text(disassemble(static_cast<Scene*>(s)->materials[slot].program), buf, cap, len);
}
void ref_scene_analysis_json(void* s, int slot, char* buf, size_t cap, size_t* len) {
    copy_text(analysis_to_json(static_cast<Scene*>(s)->materials[slot].analyzed), buf, cap, len);
}

static ShadingPoint read_sp(const float* p) {
    ShadingPoint sp;
    sp.position = v3(p);
    sp.normal = v3(p + 3);
    sp.incoming = v3(p + 6);
    sp.uv = v2(p + 9);
    sp.g1 = v2(p + 11);
    sp.g2 = v2(p + 13);
    return sp;
}

static void write_value(const Value& v, float* out) {
    const Color3 c = v.as_rgb();
    out[0] = c.r;
    out[1] = c.g;
    out[2] = c.b;
    uint32_t tag = v.is_scalar() ? 1u : 0u;
    std::memcpy(out + 3, &tag, 4);
}

// sp: 15 floats per point (position, normal, incoming, uv, g1, g2).
// values: 4 words per point (rgb + scalar tag); per-point nodes_found/instrs.
void ref_scene_execute(void* s, int slot, const float* sp, size_t n, void* cache, int mip_offset,
                       float* values, uint32_t* nodes, uint32_t* instrs) {
    const Scene& scene = *static_cast<Scene*>(s);
    CacheBinding b;
    b.cache = static_cast<MaterialCache*>(cache);
    b.mip_offset = mip_offset;
    for (size_t i = 0; i < n; ++i) {
        EvalStats st;
        const Value v = execute(scene.materials[slot].program, read_sp(sp + 15 * i), b, st);
        write_value(v, values + 4 * i);
        nodes[i] = static_cast<uint32_t>(st.nodes_found);
        instrs[i] = static_cast<uint32_t>(st.instructions_executed);
    }
}
void ref_scene_eval_reference(void* s, int slot, const float* sp, size_t n, float* values) {
    const Scene& scene = *static_cast<Scene*>(s);
    for (size_t i = 0; i < n; ++i) {
        const Value v = eval_reference(scene.materials[slot].source, read_sp(sp + 15 * i),
                                       scene.textures);
        write_value(v, values + 4 * i);
    }
}
// out per ray (24 floats): found, t, position3, normal3, uv2, slot, e1 3, e2 3, duv1 2, duv2 2, pad
void ref_scene_intersect(void* s, const float* rays, size_t n, float t_min, float t_max,
                         float* out) {
    const Scene& scene = *static_cast<Scene*>(s);
    for (size_t i = 0; i < n; ++i) {
        Ray r{v3(rays + 6 * i), v3(rays + 6 * i + 3)};
        HitRecord h;
        float* o = out + 24 * i;
        std::memset(o, 0, 24 * sizeof(float));
        if (!scene.intersect(r, t_min, t_max, &h)) continue;
        const float vals[23] = {1.0f, h.t, h.position.x, h.position.y, h.position.z, h.normal.x,
                                h.normal.y, h.normal.z, h.uv.x, h.uv.y,
                                static_cast<float>(h.material_slot), h.patch.e1.x, h.patch.e1.y,
                                h.patch.e1.z, h.patch.e2.x, h.patch.e2.y, h.patch.e2.z,
                                h.patch.duv1.x, h.patch.duv1.y, h.patch.duv2.x, h.patch.duv2.y,
                                0.0f, 0.0f};
        std::memcpy(o, vals, sizeof(vals));
    }
}
// The reference's BVH nodes (scene.cpp:154-194), 10 words each: bounds_min,
// bounds_max (float bits), left, right, first, count. Returns the node count;
// writes min(count, cap) nodes.
size_t ref_scene_bvh(void* s, uint32_t* out, size_t cap) {
    const Scene& scene = *static_cast<Scene*>(s);
    const std::vector<detail::BvhNode>& nodes = scene.*member(BvhTag{});
    for (size_t i = 0; i < nodes.size() && i < cap; ++i) {
        const detail::BvhNode& n = nodes[i];
        const float b[6] = {n.bounds_min.x, n.bounds_min.y, n.bounds_min.z,
                            n.bounds_max.x, n.bounds_max.y, n.bounds_max.z};
        std::memcpy(out + 10 * i, b, sizeof(b));
        std::memcpy(out + 10 * i + 6, &n.left, 4);
        std::memcpy(out + 10 * i + 7, &n.right, 4);
        out[10 * i + 8] = n.first;
        out[10 * i + 9] = n.count;
    }
    return nodes.size();
}
void ref_scene_occluded(void* s, const float* rays, size_t n, float t_min, const float* t_max,
                        uint8_t* out) {
    const Scene& scene = *static_cast<Scene*>(s);
    for (size_t i = 0; i < n; ++i) {
        Ray r{v3(rays + 6 * i), v3(rays + 6 * i + 3)};
        out[i] = scene.occluded(r, t_min, t_max[i]);
    }
}

// ---- restated render() ------------------------------------------------------
struct RefRenderParams {
    int32_t width, height, spp, max_bounces;
    int32_t mode;         // 0 cache off, 1 epoch-sequential (immediate inserts), 2 threaded tiles,
                          // 3 epoch-sequential deterministic (deferred, ordered inserts)
    int32_t mip_offset;
    uint64_t n_cells;
    uint32_t n_entries;
    uint32_t first_sample;
    uint64_t rng_seed;
    float diffuse_spread;
    int32_t tile_size;
    int32_t shard_rank, shard_count, shard_mode;
    int32_t threads;
    int32_t samples_per_pass;  // epoch-sequential order: (pass, bounce, sample, pixel)
};

struct RefRenderStats {
    double wall_time_s;
    uint64_t lookups, hits, inserts_won, inserts_lost_full;
    uint64_t stores_attempted, stores_won, instructions_executed;
    uint64_t paths, shading_points;
};

// ---- image I/O (image.cpp) -------------------------------------------------
static ImageF to_image(int w, int h, const float* rgb) {
    ImageF img(w, h);
    for (size_t i = 0; i < img.pixels.size(); ++i) img.pixels[i] = {rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]};
    return img;
}
int ref_write_ppm(const char* path, int w, int h, const float* rgb, int gamma) {
    try {
        write_ppm(path, to_image(w, h, rgb), gamma != 0);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}
int ref_write_pfm(const char* path, int w, int h, const float* rgb) {
    try {
        write_pfm(path, to_image(w, h, rgb));
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}
// out may be null (size query): returns width/height through w/h.
int ref_read_pfm(const char* path, int* w, int* h, float* out) {
    try {
        const ImageF img = read_pfm(path);
        *w = img.width;
        *h = img.height;
        if (out) {
            for (size_t i = 0; i < img.pixels.size(); ++i) {
                out[3 * i] = img.pixels[i].r;
                out[3 * i + 1] = img.pixels[i].g;
                out[3 * i + 2] = img.pixels[i].b;
            }
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

}  // extern "C"

namespace {

constexpr float kTMin = 1e-4f;
constexpr float kEps = 1e-4f;
constexpr float kInvPi = 0.318309886183790671538f;
constexpr float kTwoPi = 6.28318530717958647692f;

struct Cam {
    Vec3 pos, fwd, right, up;
    float tan_half, aspect, spread;
};

// Identical arithmetic to mcg_camera_setup.
Cam make_camera(const Scene& s, int w, int h) {
    Cam c;
    c.pos = s.camera.position;
    c.fwd = normalize(s.camera.look_at - s.camera.position);
    c.right = normalize(cross(c.fwd, s.camera.up));
    c.up = cross(c.right, c.fwd);
    const float vfov = s.camera.vfov_deg * (3.14159265358979323846f / 180.0f);
    c.tan_half = std::tan(vfov * 0.5f);
    c.aspect = static_cast<float>(w) / static_cast<float>(h);
    c.spread = cone_for_camera(vfov, h).spread;
    return c;
}

struct PathState {
    Ray ray;
    RayCone cone;
    Color3 thr{1, 1, 1};
    Color3 L{0, 0, 0};
    uint32_t nodes = 0;
    bool alive = true;
};

inline uint32_t dim_rect(int b, int j, int k) { return 2u + 64u * b + 2u * j + k; }
inline uint32_t dim_bounce(int b, int k) { return 2u + 64u * b + 62u + k; }

void start_path(const Cam& cam, int x, int y, int w, int h, const PathRng& rng, PathState& ps) {
    const float jx = rng.sample(0), jy = rng.sample(1);
    const float sx = ((static_cast<float>(x) + jx) / static_cast<float>(w)) * 2.0f - 1.0f;
    const float sy = 1.0f - ((static_cast<float>(y) + jy) / static_cast<float>(h)) * 2.0f;
    const float a = (sx * cam.tan_half) * cam.aspect;
    const float b = sy * cam.tan_half;
    const Vec3 d = (cam.fwd + cam.right * a) + cam.up * b;
    ps = PathState{};
    ps.ray = {cam.pos, normalize(d)};
    ps.cone = {0.0f, cam.spread};
}

struct Counters {
    uint64_t stores_attempted = 0, stores_won = 0, instructions = 0, shading_points = 0;
};

// Deterministic-insert mode (mode 3) on the reference's own code. An epoch is
// one (pass, bounce) wavefront: its lookups must read the table as it was
// when the epoch began, and its stores are applied at the epoch's end in
// (sample-in-pass, pixel, store ordinal) order with MaterialCache::update's
// semantics (cache.cpp:94-119) -- the rule mc_oracle.c (mode 3) and the GPU
// (k_shade<true> + k_apply_ordered) implement. The reference's execute()
// (stackvm.cpp:248-368) inserts immediately, so around each call:
//   before: the cells of every descriptor the program can look up at this
//           shading point (stackvm.cpp:331-340: mip_level / texel_indices of
//           the point, or the non-uv sentinel) are snapshotted;
//   after:  each slot that went 0 -> word during the call is an insert this
//           point won; it is queued as (descriptor, payload, key), the slot
//           is set back to 0 and the won-insert counter decremented, so the
//           next point sees the epoch-start table again;
//   apply:  the queue, sorted by key, goes through MaterialCache::update.
// A store that found its cell full or its key present at epoch start can
// only find the same at apply time (slots are write-once and fill as a
// prefix), so queueing the won inserts alone is exact; the lost-full
// counter of those stores is the one update() bumped during the call.
// A program with two cache points on the same node (a shared DAG node
// re-emitted per consumer, stackvm.cpp:114-118) would see its own first
// store in the immediate call; such programs are rejected (none of the
// synthetic scenes has one).
struct DeferredStore {
    CacheDescriptor desc;
    uint32_t payload;
    uint32_t key;
};

struct ProgramCachePoints {
    std::vector<uint32_t> node_idx, bracket;
    std::vector<uint8_t> uses_uv;
    std::vector<uint32_t> store_ord;   // by bracket
};

class Deferred {
public:
    Deferred(const Scene& scene, MaterialCache* cache) : cache_(cache) {
        table_ = (cache->*member(TableTag{})).get();
        for (const auto& m : scene.materials) {
            ProgramCachePoints pc;
            pc.store_ord.assign(kMaxCachePoints, 0);
            uint32_t stores = 0;
            for (const Instruction& ins : m.program.code) {
                if (ins.op == Opcode::CacheLookup) {
                    for (uint32_t n : pc.node_idx) {
                        if (n == ins.node_idx) {
                            throw std::runtime_error("deferred mode: a program has two cache points on node " +
                                                     std::to_string(n));
                        }
                    }
                    pc.node_idx.push_back(ins.node_idx);
                    pc.bracket.push_back(ins.bracket);
                    pc.uses_uv.push_back(ins.uses_uv ? 1 : 0);
                } else if (ins.op == Opcode::CacheStore) {
                    pc.store_ord.at(ins.bracket) = stores++;
                }
            }
            points_.push_back(std::move(pc));
        }
    }

    uint32_t key_base = 0;

    void before(const CompiledProgram& prog, uint32_t slot, const ShadingPoint& sp, int mip_offset) {
        const ProgramCachePoints& pc = points_[slot];
        const uint64_t nc = cache_->n_cells();
        const uint32_t ne = cache_->n_entries();
        descs_.clear();
        cells_.clear();
        ords_.clear();
        snap_.clear();
        snap_cells_.clear();
        for (size_t k = 0; k < pc.node_idx.size(); ++k) {
            CacheDescriptor d;
            d.mat_idx = prog.material_id;
            d.node_idx = pc.node_idx[k];
            if (pc.uses_uv[k]) {
                d.mip_level = mip_level(sp.g1, sp.g2, mip_offset);
                const auto [tx, ty] = texel_indices(sp.uv, d.mip_level);
                d.texel_x = tx;
                d.texel_y = ty;
            }
            const uint64_t cell = hash_cell(d) % nc;
            descs_.push_back(d);
            cells_.push_back(cell);
            ords_.push_back(pc.store_ord[pc.bracket[k]]);
            bool seen = false;
            for (uint64_t c : snap_cells_) seen = seen || c == cell;
            if (seen) continue;
            snap_cells_.push_back(cell);
            for (uint32_t e = 0; e < ne; ++e) snap_.push_back(table_[cell * ne + e].load());
        }
    }

    void after() {
        const uint32_t ne = cache_->n_entries();
        uint64_t taken = 0;
        for (size_t c = 0; c < snap_cells_.size(); ++c) {
            const uint64_t cell = snap_cells_[c];
            for (uint32_t e = 0; e < ne; ++e) {
                const uint64_t now = table_[cell * ne + e].load();
                const uint64_t was = snap_[c * ne + e];
                if (now == was) continue;
                if (was != 0) throw std::runtime_error("deferred mode: an occupied slot changed");
                size_t k = 0;
                while (k < descs_.size() && !(cells_[k] == cell && hash_check(descs_[k]) == entry_hash(now))) ++k;
                if (k == descs_.size()) throw std::runtime_error("deferred mode: insert of an unknown key");
                queue_.push_back({descs_[k], entry_payload(now), key_base | ords_[k]});
                table_[cell * ne + e].store(0);
                ++taken;
            }
        }
        (cache_->*member(WonTag{})).fetch_sub(taken);
    }

    // Epoch end: the queued stores in key order through update(). Returns
    // the number of inserts won.
    uint64_t apply() {
        std::sort(queue_.begin(), queue_.end(),
                  [](const DeferredStore& a, const DeferredStore& b) { return a.key < b.key; });
        uint64_t won = 0;
        for (const DeferredStore& q : queue_) {
            const UpdateResult r = cache_->update(q.desc, decode_value(q.payload));
            if (r.outcome == InsertOutcome::Won) {
                if (entry_payload(r.packed) != q.payload) throw std::runtime_error("deferred mode: payload round trip");
                ++won;
            }
        }
        queue_.clear();
        return won;
    }

private:
    MaterialCache* cache_;
    std::atomic<uint64_t>* table_;
    std::vector<ProgramCachePoints> points_;
    std::vector<CacheDescriptor> descs_;
    std::vector<uint64_t> cells_, snap_, snap_cells_;
    std::vector<uint32_t> ords_;
    std::vector<DeferredStore> queue_;
};

// One path vertex: intersect, shade, next-event estimation, bounce.
void path_vertex(const Scene& scene, const RefRenderParams& p, const CacheBinding& binding,
                 const PathRng& rng, int b, PathState& ps, Counters& cnt, Deferred* dq = nullptr) {
    HitRecord hit;
    if (!scene.intersect(ps.ray, kTMin, INFINITY, &hit)) {
        ps.L = ps.L + ps.thr * scene.env;
        ps.alive = false;
        return;
    }
    ps.cone = propagate(ps.cone, hit.t);
    const auto [g1, g2] = footprint_gradients(ps.cone, ps.ray.dir, hit.normal, hit.patch);
    ShadingPoint sp{hit.position, hit.normal, ps.ray.dir, hit.uv, g1, g2};
    EvalStats st;
    const CompiledProgram& prog = scene.materials[hit.material_slot].program;
    if (dq) dq->before(prog, hit.material_slot, sp, binding.mip_offset);
    const Value v = execute(prog, sp, binding, st);
    if (dq) dq->after();
    ++cnt.shading_points;
    cnt.stores_attempted += st.stores_attempted;
    if (!dq) cnt.stores_won += st.stores_won;   // deferred: counted at the epoch's apply
    cnt.instructions += st.instructions_executed;
    ps.nodes += static_cast<uint32_t>(st.nodes_found);
    const Color3 c = v.as_rgb();
    const Color3 alb{std::fmin(std::fmax(c.r, 0.0f), 1.0f), std::fmin(std::fmax(c.g, 0.0f), 1.0f),
                     std::fmin(std::fmax(c.b, 0.0f), 1.0f)};
    const Color3 f = alb * kInvPi;
    const Color3 tf = ps.thr * f;
    const Vec3 n = hit.normal;
    const Vec3 o = hit.position + n * kEps;
    for (const PointLight& l : scene.point_lights) {
        const Vec3 toL = l.position - o;
        const float d2 = dot(toL, toL);
        const float dist = std::sqrt(d2);
        const Vec3 wi = toL * (1.0f / dist);
        const float cs = dot(n, wi);
        if (cs > 0.0f && !scene.occluded({o, wi}, kTMin, dist)) {
            const float w = cs / d2;
            ps.L = ps.L + tf * (l.intensity * w);
        }
    }
    for (size_t j = 0; j < scene.rect_lights.size(); ++j) {
        const RectLight& l = scene.rect_lights[j];
        const float u = rng.sample(dim_rect(b, static_cast<int>(j), 0));
        const float vv = rng.sample(dim_rect(b, static_cast<int>(j), 1));
        const Vec3 pl = (l.corner + l.edge_u * u) + l.edge_v * vv;
        const Vec3 nl = cross(l.edge_u, l.edge_v);
        const float area = length(nl);
        const Vec3 toL = pl - o;
        const float d2 = dot(toL, toL);
        const float dist = std::sqrt(d2);
        const Vec3 wi = toL * (1.0f / dist);
        const float cs = dot(n, wi);
        const float cl = std::fabs(dot(nl, wi)) / area;
        if (cs > 0.0f && cl > 0.0f && !scene.occluded({o, wi}, kTMin, dist)) {
            const float w = ((cs * cl) * area) / d2;
            ps.L = ps.L + tf * (l.radiance * w);
        }
    }
    if (b == p.max_bounces) {
        ps.alive = false;
        return;
    }
    const float r1 = rng.sample(dim_bounce(b, 0));
    const float r2 = rng.sample(dim_bounce(b, 1));
    float sphi, cphi;
    mc_sincosf(r1 * kTwoPi, &sphi, &cphi);
    const float r = std::sqrt(r2);
    const float lx = r * cphi, ly = r * sphi;
    const float lz = std::sqrt(std::fmax(0.0f, 1.0f - r2));
    const float sign = std::copysign(1.0f, n.z);
    const float a = -1.0f / (sign + n.z);
    const float bb = (n.x * n.y) * a;
    const Vec3 t{1.0f + ((sign * n.x) * n.x) * a, sign * bb, -sign * n.x};
    const Vec3 bt{bb, sign + ((n.y * n.y) * a), -n.y};
    const Vec3 nd = normalize((t * lx + bt * ly) + n * lz);
    ps.thr = ps.thr * alb;
    ps.cone = widen(ps.cone, p.diffuse_spread);
    ps.ray = {o, nd};
}

bool tile_mine(const RefRenderParams& p, int tile, int n_tiles) {
    if (p.shard_count <= 1) return true;
    if (p.shard_mode == 0) return tile % p.shard_count == p.shard_rank;
    const int lo = static_cast<int>(static_cast<int64_t>(n_tiles) * p.shard_rank / p.shard_count);
    const int hi =
        static_cast<int>(static_cast<int64_t>(n_tiles) * (p.shard_rank + 1) / p.shard_count);
    return tile >= lo && tile < hi;
}

}  // namespace

extern "C" int ref_render(void* s, const RefRenderParams* pp, void* external_cache,
                          double* radiance, double* nodes_found, uint32_t* samples,
                          uint64_t* hits_per_sample, RefRenderStats* stats) {
    return guard([&] {
        const Scene& scene = *static_cast<Scene*>(s);
        RefRenderParams p = *pp;
        const int w = p.width ? p.width : scene.camera.width;
        const int h = p.height ? p.height : scene.camera.height;
        const Cam cam = make_camera(scene, w, h);
        std::unique_ptr<MaterialCache> own;
        MaterialCache* cache = nullptr;
        if (p.mode != 0) {
            cache = static_cast<MaterialCache*>(external_cache);
            if (!cache) {
                own = std::make_unique<MaterialCache>(p.n_cells, p.n_entries);
                cache = own.get();
            }
        }
        CacheBinding binding;
        binding.cache = cache;
        binding.mip_offset = p.mip_offset;
        const int ts = p.tile_size > 0 ? p.tile_size : 16;
        const int tiles_x = (w + ts - 1) / ts, tiles_y = (h + ts - 1) / ts;
        const int n_tiles = tiles_x * tiles_y;
        std::vector<uint32_t> pixels;  // this shard's pixels, ascending index
        for (int y = 0; y < h; ++y) {
            for (int x = 0; x < w; ++x) {
                if (tile_mine(p, (y / ts) * tiles_x + x / ts, n_tiles)) {
                    pixels.push_back(static_cast<uint32_t>(y * w + x));
                }
            }
        }
        if (cache) cache->reset_counters();
        const auto t0 = std::chrono::steady_clock::now();
        Counters total;
        uint64_t paths = 0;
        if (p.mode != 2) {
            // Epoch order: pass of k samples, bounce b, sample, pixel ascending
            // (the GPU wavefront order). Mode 1: inserts are immediate; mode
            // 3: deferred to the epoch's end (class Deferred).
            const int k = p.samples_per_pass > 0 ? std::min(p.samples_per_pass, p.spp) : 1;
            const size_t np = pixels.size();
            std::unique_ptr<Deferred> dq;
            if (p.mode == 3) dq = std::make_unique<Deferred>(scene, cache);
            const uint32_t wh = static_cast<uint32_t>(w) * static_cast<uint32_t>(h);
            std::vector<PathState> st(np * static_cast<size_t>(k));
            for (int start = 0; start < p.spp; start += k) {
                const int kk = std::min(k, p.spp - start);
                for (int j = 0; j < kk; ++j) {
                    for (size_t q = 0; q < np; ++q) {
                        const uint32_t pix = pixels[q];
                        start_path(cam, pix % w, pix / w, w, h,
                                   PathRng(p.rng_seed, pix, p.first_sample + start + j),
                                   st[j * np + q]);
                    }
                }
                for (int b = 0; b <= p.max_bounces; ++b) {
                    for (int j = 0; j < kk; ++j) {
                        for (size_t q = 0; q < np; ++q) {
                            PathState& ps = st[j * np + q];
                            if (!ps.alive) continue;
                            if (dq) dq->key_base = (static_cast<uint32_t>(j) * wh + pixels[q]) << 6;
                            path_vertex(scene, p, binding,
                                        PathRng(p.rng_seed, pixels[q], p.first_sample + start + j),
                                        b, ps, total, dq.get());
                        }
                    }
                    if (dq) total.stores_won += dq->apply();
                }
                for (size_t q = 0; q < np; ++q) {
                    for (int j = 0; j < kk; ++j) {
                        const PathState& ps = st[j * np + q];
                        const uint32_t pix = pixels[q];
                        radiance[3 * pix] += ps.L.r;
                        radiance[3 * pix + 1] += ps.L.g;
                        radiance[3 * pix + 2] += ps.L.b;
                        nodes_found[pix] += ps.nodes;
                        samples[pix] += 1;
                        if (hits_per_sample) hits_per_sample[start + j] += ps.nodes;
                    }
                }
                paths += np * kk;
            }
        } else {
            // Tile queue over worker threads: the reference
            // CPU path's own execution model, nondeterministic with a cache.
            const int nthreads = p.threads > 0 ? p.threads
                                               : static_cast<int>(std::thread::hardware_concurrency());
            std::vector<int> tiles;
            for (int t = 0; t < n_tiles; ++t) if (tile_mine(p, t, n_tiles)) tiles.push_back(t);
            std::atomic<size_t> next{0};
            std::mutex mu;
            std::vector<uint64_t> hps(p.spp, 0);
            auto worker = [&] {
                Counters local;
                std::vector<uint64_t> lh(p.spp, 0);
                for (;;) {
                    const size_t ti = next.fetch_add(1);
                    if (ti >= tiles.size()) break;
                    const int tx = tiles[ti] % tiles_x, ty = tiles[ti] / tiles_x;
                    for (int y = ty * ts; y < std::min(h, (ty + 1) * ts); ++y) {
                        for (int x = tx * ts; x < std::min(w, (tx + 1) * ts); ++x) {
                            const uint32_t pix = static_cast<uint32_t>(y * w + x);
                            for (int si = 0; si < p.spp; ++si) {
                                const PathRng rng(p.rng_seed, pix, p.first_sample + si);
                                PathState ps;
                                start_path(cam, x, y, w, h, rng, ps);
                                for (int b = 0; b <= p.max_bounces && ps.alive; ++b) {
                                    path_vertex(scene, p, binding, rng, b, ps, local);
                                }
                                radiance[3 * pix] += ps.L.r;
                                radiance[3 * pix + 1] += ps.L.g;
                                radiance[3 * pix + 2] += ps.L.b;
                                nodes_found[pix] += ps.nodes;
                                samples[pix] += 1;
                                lh[si] += ps.nodes;
                            }
                        }
                    }
                }
                std::lock_guard<std::mutex> lk(mu);
                total.stores_attempted += local.stores_attempted;
                total.stores_won += local.stores_won;
                total.instructions += local.instructions;
                total.shading_points += local.shading_points;
                for (int si = 0; si < p.spp; ++si) hps[si] += lh[si];
            };
            std::vector<std::thread> pool;
            for (int i = 0; i < nthreads; ++i) pool.emplace_back(worker);
            for (auto& t : pool) t.join();
            if (hits_per_sample) for (int si = 0; si < p.spp; ++si) hits_per_sample[si] += hps[si];
            paths = static_cast<uint64_t>(pixels.size()) * p.spp;
        }
        const auto t1 = std::chrono::steady_clock::now();
        if (stats) {
            std::memset(stats, 0, sizeof(*stats));
            stats->wall_time_s = std::chrono::duration<double>(t1 - t0).count();
            if (cache) {
                const auto k = cache->counters();
                stats->lookups = k.lookups;
                stats->hits = k.hits;
                stats->inserts_won = k.inserts_won;
                stats->inserts_lost_full = k.inserts_lost_full;
            }
            stats->stores_attempted = total.stores_attempted;
            stats->stores_won = total.stores_won;
            stats->instructions_executed = total.instructions;
            stats->paths = paths;
            stats->shading_points = total.shading_points;
        }
    });
}

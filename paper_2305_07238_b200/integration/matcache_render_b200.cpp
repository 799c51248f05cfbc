// matcache_render_b200.cpp — the link-level drop-in for the reference's C++
// renderer API. The reference declares render() and the experiment helpers in
// include/matcache/tracer.hpp:69-92 but ships no definition (src/tracer.cpp is
// absent, proj/core/CMakeLists.txt:14). Linking this file plus libmcg.so into
// matcache_core provides them, backed by the B200 kernels behind the C ABI
// (include/mcg.h). Build: see INTEGRATION.md (and oracle/Makefile `dropin`,
// which compiles it against the reference headers in place for the tests).
//
// What it does per call:
//   Scene (scene.hpp:91-123) + compiled programs (stackvm.hpp:73-79)
//     -> mcg_scene_in (meshes, spheres, lights, camera, flattened bytecode,
//        RGBA textures) -> mcg_scene_build (BVH rebuilt with the reference's
//        median split, scene.cpp:154-194) -> mcg_upload_scene -> mcg_render.
// Status codes are rethrown as the reference's exception types.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <sstream>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "matcache/tracer.hpp"
#include "matcache_render_b200.hpp"
#include "mcg.h"

namespace matcache {
namespace {

[[noreturn]] void rethrow(mcg_status s) {
    const std::string msg = mcg_last_error();
    switch (s) {
        case MCG_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case MCG_ERR_OVERFLOW: throw std::overflow_error(msg);
        case MCG_ERR_GRAPH: throw GraphError(msg);
        case MCG_ERR_COMPILE: throw CompileError(msg);
        case MCG_ERR_SCENE: throw SceneError(msg);
        case MCG_ERR_IMAGE_IO: throw ImageIoError(msg);
        default: throw std::runtime_error(msg);
    }
}

void ok(mcg_status s) {
    if (s != MCG_OK) rethrow(s);
}

// Device contexts, one set per process (the reference render() is
// synchronous). `ctx` is device 0 alone (external-cache renders: the caller's
// table is one table); `multi` spans every GPU the process may use
// (MATCACHE_B200_DEVICES="0,1,..." or all visible ones): render() without an
// external cache deals its tiles to all of them with a cache replica each
// and gathers the frame over NCCL, as the reference's render() uses every
// worker thread (tracer.hpp:12, 69-70).
struct Device {
    std::mutex mu;
    mcg_ctx* ctx = nullptr;
    mcg_ctx* multi = nullptr;
    // The scene, identified by content (a fingerprint of everything the
    // devices receive), never by the Scene's address: a different or edited
    // Scene at the same address must not render with stale data.
    uint64_t scene_fp = 0;
    uint64_t uploaded_fp = 0, multi_fp = 0;   // what each context holds
    mcg_scene* scene = nullptr;
    // Device tables standing in for external MaterialCache objects, reused
    // across calls (an 800 MB allocation is not free). The host table stays
    // the truth: every call seeds the device table from its slot words and
    // replays the render's won inserts back through update() (table_for /
    // sync_back), so a table reused at a recycled address, or changed by the
    // caller between renders, is never stale.
    std::map<const MaterialCache*, mcg_cache*> tables;
};

Device& device() {
    static Device d;
    return d;
}

uint8_t flags_of(const Instruction& ins) {
    uint8_t f = 0;
    if (ins.uses_uv) f |= MCG_F_USES_UV;
    if (ins.scalar_result) f |= MCG_F_SCALAR_RESULT;
    if (ins.op == Opcode::TexSample && ins.wrap == WrapMode::Clamp) f |= MCG_F_WRAP_CLAMP;
    if (ins.op == Opcode::LoadUv) f |= static_cast<uint8_t>(static_cast<unsigned>(ins.uv_channel) << MCG_F_UV_SHIFT);
    return f;
}

struct Flattened {
    std::vector<mcg_program> programs;
    std::vector<mcg_insn> code;
    std::vector<mcg_const> consts;
    std::vector<mcg_noise> noise;
    std::vector<mcg_ramp> ramps;
    std::vector<mcg_ramp_stop> stops;
    std::vector<mcg_texture> textures;
    std::vector<float> texels;
    std::unordered_map<const Texture*, uint32_t> tex_id;
};

uint32_t texture_id(Flattened& F, const Texture* t) {
    const auto it = F.tex_id.find(t);
    if (it != F.tex_id.end()) return it->second;
    const uint32_t id = static_cast<uint32_t>(F.textures.size());
    F.textures.push_back({t->image.width, t->image.height, F.texels.size() / 4});
    for (const Color3& c : t->image.pixels) {
        F.texels.insert(F.texels.end(), {c.r, c.g, c.b, 0.0f});
    }
    F.tex_id.emplace(t, id);
    return id;
}

// CompiledProgram (stackvm.hpp:73-79) -> device instruction words + pools.
void flatten(Flattened& F, const CompiledProgram& prog) {
    mcg_program p{};
    p.material_id = prog.material_id;
    p.code_offset = static_cast<uint32_t>(F.code.size());
    p.code_len = static_cast<uint32_t>(prog.code.size());
    p.cache_point_count = prog.cache_point_count;
    const uint32_t ramp_base = static_cast<uint32_t>(F.ramps.size());
    for (const auto& stops : prog.ramps) {
        F.ramps.push_back({static_cast<uint32_t>(F.stops.size()), static_cast<uint32_t>(stops.size())});
        for (const auto& s : stops) F.stops.push_back({s.t, s.color.r, s.color.g, s.color.b});
    }
    for (const Instruction& ins : prog.code) {
        mcg_insn w{};
        w.op = static_cast<uint8_t>(ins.op);
        w.flags = flags_of(ins);
        w.bracket = static_cast<uint16_t>(ins.bracket);
        switch (ins.op) {
            case Opcode::PushConst: {
                const Color3 c = ins.constant.as_rgb();
                w.arg = static_cast<uint32_t>(F.consts.size());
                F.consts.push_back({{c.r, c.g, c.b}, ins.constant.is_scalar() ? 1u : 0u});
                break;
            }
            case Opcode::TexSample: w.arg = texture_id(F, ins.texture); break;
            case Opcode::Checker: w.imm.f = ins.checker_scale; break;
            case Opcode::Noise:
                w.arg = static_cast<uint32_t>(F.noise.size());
                F.noise.push_back({ins.noise.octaves, ins.noise.frequency, ins.noise.lacunarity,
                                   ins.noise.gain});
                break;
            case Opcode::Ramp: w.arg = ramp_base + ins.ramp_index; break;
            case Opcode::CacheLookup:
                w.arg = ins.node_idx;
                w.imm.i = ins.skip_offset;
                break;
            case Opcode::CacheStore: w.arg = ins.node_idx; break;
            default: break;
        }
        F.code.push_back(w);
    }
    uint32_t max_stack = 0;
    ok(mcg_schedule_program(F.code.data() + p.code_offset, p.code_len, F.consts.data(),
                            static_cast<uint32_t>(F.consts.size()), &max_stack));
    p.max_stack = max_stack;
    F.programs.push_back(p);
}

// Everything mcg_scene_build receives, owned (the mcg_scene_in points into it).
struct SceneInput {
    Flattened F;
    std::vector<mcg_mesh_in> meshes;
    std::vector<std::vector<float>> pos, uvs;
    std::vector<mcg_sphere_in> spheres;
    std::vector<mcg_point_light> pl;
    std::vector<mcg_rect_light> rl;
    mcg_scene_in in{};
};

// FNV-1a over bytes, folded through a splitmix64 finalizer per array.
struct Fingerprint {
    uint64_t h = 0xcbf29ce484222325ull;
    void bytes(const void* p, size_t n) {
        const unsigned char* b = static_cast<const unsigned char*>(p);
        uint64_t x = 0xcbf29ce484222325ull;
        for (size_t i = 0; i < n; ++i) x = (x ^ b[i]) * 0x100000001b3ull;
        x ^= n;
        x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
        x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
        h = (h ^ x ^ (x >> 31)) * 0x100000001b3ull;
    }
    template <typename T>
    void vec(const std::vector<T>& v) { bytes(v.data(), v.size() * sizeof(T)); }
};

uint64_t fingerprint(const SceneInput& S) {
    Fingerprint f;
    const mcg_scene_in& in = S.in;
    f.bytes(in.cam_position, sizeof(in.cam_position));
    f.bytes(in.cam_look_at, sizeof(in.cam_look_at));
    f.bytes(in.cam_up, sizeof(in.cam_up));
    f.bytes(&in.cam_vfov_deg, sizeof(in.cam_vfov_deg));
    f.bytes(&in.cam_width, sizeof(in.cam_width));
    f.bytes(&in.cam_height, sizeof(in.cam_height));
    f.bytes(in.env, sizeof(in.env));
    for (size_t i = 0; i < S.meshes.size(); ++i) {
        f.vec(S.pos[i]);
        f.vec(S.uvs[i]);
        f.bytes(S.meshes[i].indices, S.meshes[i].n_indices * sizeof(uint32_t));
        f.bytes(&S.meshes[i].material_id, sizeof(uint32_t));
    }
    f.vec(S.spheres);
    f.vec(S.pl);
    f.vec(S.rl);
    f.vec(S.F.programs);
    f.vec(S.F.code);
    f.vec(S.F.consts);
    f.vec(S.F.noise);
    f.vec(S.F.ramps);
    f.vec(S.F.stops);
    f.vec(S.F.textures);
    f.vec(S.F.texels);
    return f.h;
}

void scene_input(const Scene& scene, SceneInput& S) {
    Flattened& F = S.F;
    for (const MaterialRuntime& m : scene.materials) flatten(F, m.program);
    std::vector<mcg_mesh_in>& meshes = S.meshes;
    std::vector<std::vector<float>>& pos = S.pos;
    std::vector<std::vector<float>>& uvs = S.uvs;
    pos.assign(scene.meshes.size(), {});
    uvs.assign(scene.meshes.size(), {});
    for (size_t i = 0; i < scene.meshes.size(); ++i) {
        const MeshObject& m = scene.meshes[i];
        for (const Vec3& p : m.positions) pos[i].insert(pos[i].end(), {p.x, p.y, p.z});
        for (const Vec2& t : m.uvs) uvs[i].insert(uvs[i].end(), {t.x, t.y});
        if (m.positions.size() != m.uvs.size()) throw SceneError("mesh must carry one uv per vertex");
        meshes.push_back({static_cast<uint32_t>(m.positions.size()),
                          static_cast<uint32_t>(m.indices.size()), m.material_id, pos[i].data(),
                          uvs[i].data(), m.indices.data()});
    }
    std::vector<mcg_sphere_in>& spheres = S.spheres;
    for (const SphereObject& s : scene.spheres) {
        spheres.push_back({{s.center.x, s.center.y, s.center.z}, s.radius, s.material_id});
    }
    std::vector<mcg_point_light>& pl = S.pl;
    for (const PointLight& l : scene.point_lights) {
        pl.push_back({{l.position.x, l.position.y, l.position.z},
                      {l.intensity.r, l.intensity.g, l.intensity.b}});
    }
    std::vector<mcg_rect_light>& rl = S.rl;
    for (const RectLight& l : scene.rect_lights) {
        rl.push_back({{l.corner.x, l.corner.y, l.corner.z}, {l.edge_u.x, l.edge_u.y, l.edge_u.z},
                      {l.edge_v.x, l.edge_v.y, l.edge_v.z}, {l.radiance.r, l.radiance.g, l.radiance.b}});
    }
    mcg_scene_in& in = S.in;
    const Camera& c = scene.camera;
    const float cam[9] = {c.position.x, c.position.y, c.position.z, c.look_at.x, c.look_at.y,
                          c.look_at.z, c.up.x, c.up.y, c.up.z};
    std::memcpy(in.cam_position, cam, sizeof(in.cam_position));
    std::memcpy(in.cam_look_at, cam + 3, sizeof(in.cam_look_at));
    std::memcpy(in.cam_up, cam + 6, sizeof(in.cam_up));
    in.cam_vfov_deg = c.vfov_deg;
    in.cam_width = c.width;
    in.cam_height = c.height;
    in.env[0] = scene.env.r;
    in.env[1] = scene.env.g;
    in.env[2] = scene.env.b;
    in.n_meshes = static_cast<uint32_t>(meshes.size());
    in.meshes = meshes.data();
    in.n_spheres = static_cast<uint32_t>(spheres.size());
    in.spheres = spheres.data();
    in.n_point_lights = static_cast<uint32_t>(pl.size());
    in.point_lights = pl.data();
    in.n_rect_lights = static_cast<uint32_t>(rl.size());
    in.rect_lights = rl.data();
    in.n_programs = static_cast<uint32_t>(F.programs.size());
    in.programs = F.programs.data();
    in.n_code = static_cast<uint32_t>(F.code.size());
    in.code = F.code.data();
    in.n_consts = static_cast<uint32_t>(F.consts.size());
    in.consts = F.consts.data();
    in.n_noise = static_cast<uint32_t>(F.noise.size());
    in.noise = F.noise.data();
    in.n_ramps = static_cast<uint32_t>(F.ramps.size());
    in.ramps = F.ramps.data();
    in.n_ramp_stops = static_cast<uint32_t>(F.stops.size());
    in.ramp_stops = F.stops.data();
    in.n_textures = static_cast<uint32_t>(F.textures.size());
    in.textures = F.textures.data();
    in.n_texels = F.texels.size() / 4;
    in.texels = F.texels.data();
}

// The device table standing in for `ext` for one call: (re)created when the
// shape differs, then seeded with the host table's slot words
// (cache.hpp:83-86) so it holds exactly what `ext` holds; the won-insert log
// records what this render adds. Returns the log capacity (the empty slots:
// a table can win no more inserts than that).
uint64_t table_for(Device& D, MaterialCache* ext, mcg_cache** out) {
    mcg_cache*& t = D.tables[ext];
    if (t) {
        uint64_t nc = 0;
        uint32_t ne = 0;
        ok(mcg_cache_shape(t, &nc, &ne));
        if (nc != ext->n_cells() || ne != ext->n_entries()) {
            mcg_cache_destroy(t);
            t = nullptr;
        }
    }
    if (!t) ok(mcg_cache_create(D.ctx, ext->n_cells(), ext->n_entries(), &t));
    const uint64_t total = ext->slot_count();
    const uint64_t chunk = 1ull << 22;
    std::vector<uint64_t> words(static_cast<size_t>(std::min(total, chunk)));
    uint64_t occupied = 0;
    for (uint64_t first = 0; first < total; first += chunk) {
        const uint64_t n = std::min(chunk, total - first);
        for (uint64_t i = 0; i < n; ++i) {
            words[i] = ext->slot_word(first + i);
            occupied += words[i] != 0;
        }
        ok(mcg_cache_write_slots(t, first, static_cast<size_t>(n), words.data()));
    }
    ok(mcg_cache_counters_reset(t));
    const uint64_t cap = std::max<uint64_t>(1, total - occupied);
    ok(mcg_cache_insert_log_start(t, cap));
    *out = t;
    return cap;
}

// After the render: the device's won inserts, replayed through the caller's
// MaterialCache::update (cache.cpp:94-119) in (cell, entry) order -- each
// lands in its cell's first empty slot, i.e. exactly the device's slot, so
// the host table, its inserts_won counter, occupied_slots() and dump()
// match what a reference render into `ext` would leave behind in shape (the
// lookups/hits counters have no public writer and stay the caller's).
void sync_back(mcg_cache* t, MaterialCache* ext, uint64_t cap) {
    uint64_t won = 0;
    ok(mcg_cache_insert_log_stop(t, &won));
    if (won > cap) throw std::runtime_error("render(): device insert log overflow");
    std::vector<mcg_insert_record> rec(static_cast<size_t>(won));
    ok(mcg_cache_insert_log_read(t, 0, rec.size(), rec.data()));
    std::vector<std::pair<uint64_t, size_t>> order(rec.size());
    const uint64_t nc = ext->n_cells();
    const uint32_t ne = ext->n_entries();
    for (size_t i = 0; i < rec.size(); ++i) {
        order[i] = {(mcg_hash_cell(&rec[i].desc) % nc) * ne + rec[i].entry, i};
    }
    std::sort(order.begin(), order.end());
    for (const auto& [slot, i] : order) {
        const mcg_insert_record& r = rec[i];
        CacheDescriptor d;
        d.mat_idx = r.desc.mat_idx;
        d.node_idx = r.desc.node_idx;
        d.mip_level = r.desc.mip_level;
        d.texel_x = r.desc.texel_x;
        d.texel_y = r.desc.texel_y;
        const UpdateResult u = ext->update(d, decode_value(r.payload));
        if (u.outcome != InsertOutcome::Won || u.slot != slot || entry_payload(u.packed) != r.payload) {
            throw std::runtime_error("render(): host replay of the device's inserts diverged "
                                     "(external cache changed during the render?)");
        }
    }
}

}  // namespace

// Frees the device table standing in for `cache` (tables otherwise live, and
// are reused, for the process's lifetime). Declared in
// integration/matcache_render_b200.hpp.
void b200_release_cache(const MaterialCache* cache) {
    Device& D = device();
    std::lock_guard<std::mutex> lock(D.mu);
    const auto it = D.tables.find(cache);
    if (it == D.tables.end()) return;
    mcg_cache_destroy(it->second);
    D.tables.erase(it);
}

RenderResult render(const Scene& scene, const RenderConfig& config, MaterialCache* external_cache) {
    Device& D = device();
    std::lock_guard<std::mutex> lock(D.mu);
    const auto t0 = std::chrono::steady_clock::now();
    const bool use_multi = !(config.cache_enabled && external_cache);
    if (!D.ctx) {
        mcg_options opt{0, 0, nullptr, 0, nullptr};
        ok(mcg_create(&opt, &D.ctx));
        std::vector<int32_t> devs;
        if (const char* env = std::getenv("MATCACHE_B200_DEVICES")) {
            std::stringstream ss(env);
            std::string tok;
            while (std::getline(ss, tok, ',')) {
                if (!tok.empty()) devs.push_back(static_cast<int32_t>(std::stoi(tok)));
            }
        } else {
            int32_t n = 1;
            ok(mcg_device_count(&n));
            for (int32_t k = 0; k < n; ++k) devs.push_back(k);
        }
        if (devs.size() > 1) {
            mcg_options mo{devs[0], 0, nullptr, static_cast<int32_t>(devs.size()), devs.data()};
            ok(mcg_create(&mo, &D.multi));
        }
    }
    mcg_ctx* ctx = (use_multi && D.multi) ? D.multi : D.ctx;
    {
        SceneInput S;
        scene_input(scene, S);
        const uint64_t fp = fingerprint(S);
        if (!D.scene || fp != D.scene_fp) {
            if (D.scene) mcg_scene_destroy(D.scene);
            D.scene = nullptr;
            D.scene_fp = D.uploaded_fp = D.multi_fp = 0;
            ok(mcg_scene_build(&S.in, &D.scene));
            D.scene_fp = fp;
        }
        uint64_t& have = ctx == D.multi ? D.multi_fp : D.uploaded_fp;
        if (have != fp) {
            have = 0;
            ok(mcg_upload_scene(ctx, D.scene));
            have = fp;
        }
    }
    const int w = config.width ? config.width : scene.camera.width;
    const int h = config.height ? config.height : scene.camera.height;
    RenderResult result;
    result.frame = FrameBuffers(w, h);
    mcg_render_params p{};
    p.width = w;
    p.height = h;
    p.spp = config.spp;
    p.max_bounces = config.max_bounces;
    p.cache_mode = config.cache_enabled ? MCG_CACHE_CONCURRENT : MCG_CACHE_OFF;
    p.mip_offset = config.mip_offset;
    p.n_cells = config.n_cells;
    p.n_entries = config.n_entries;
    p.rng_seed = config.rng_seed;
    p.diffuse_spread = config.diffuse_spread;
    p.tile_size = config.tile_size;
    p.shard_count = 1;
    mcg_cache* table = nullptr;
    uint64_t log_cap = 0;
    if (config.cache_enabled && external_cache) log_cap = table_for(D, external_cache, &table);
    mcg_frame frame{result.frame.radiance.data(), result.frame.nodes_found.data(),
                    result.frame.samples.data()};
    std::vector<uint64_t> hps(static_cast<size_t>(std::max(config.spp, 0)), 0);
    mcg_render_stats st{};
    st.hits_per_sample = hps.data();
    ok(mcg_render(ctx, &p, table, &frame, &st));
    if (table) sync_back(table, external_cache, log_cap);
    RenderStats& rs = result.stats;
    rs.lookups = st.lookups;
    rs.hits = st.hits;
    rs.hit_rate = st.lookups ? static_cast<double>(st.hits) / static_cast<double>(st.lookups) : 0.0;
    rs.inserts_won = st.inserts_won;
    rs.inserts_lost_full = st.inserts_lost_full;
    rs.stores_attempted = st.stores_attempted;
    rs.instructions_executed = st.instructions_executed;
    rs.hits_per_sample = std::move(hps);
    rs.wall_time_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return result;
}

// ---- FrameBuffers helpers and experiment outputs (tracer.hpp:24-92) --------

ImageF FrameBuffers::radiance_image() const {
    ImageF img(width, height);
    for (size_t i = 0; i < img.pixels.size(); ++i) {
        const double n = samples[i] ? static_cast<double>(samples[i]) : 1.0;
        img.pixels[i] = {static_cast<float>(radiance[3 * i] / n),
                         static_cast<float>(radiance[3 * i + 1] / n),
                         static_cast<float>(radiance[3 * i + 2] / n)};
    }
    return img;
}

std::vector<float> FrameBuffers::nodes_found_avg() const {
    std::vector<float> out(nodes_found.size());
    for (size_t i = 0; i < out.size(); ++i) {
        out[i] = static_cast<float>(nodes_found[i] / (samples[i] ? samples[i] : 1u));
    }
    return out;
}

Color3 FrameBuffers::mean_radiance() const {
    const ImageF img = radiance_image();
    double r = 0, g = 0, b = 0;
    for (const Color3& c : img.pixels) {
        r += c.r;
        g += c.g;
        b += c.b;
    }
    const double n = img.pixels.empty() ? 1.0 : static_cast<double>(img.pixels.size());
    return {static_cast<float>(r / n), static_cast<float>(g / n), static_cast<float>(b / n)};
}

DiffStats image_error(const ImageF& a, const ImageF& b, float scale) {
    if (a.width != b.width || a.height != b.height) {
        throw std::invalid_argument("image_error: resolution mismatch");
    }
    DiffStats d;
    d.diff = ImageF(a.width, a.height);
    double sum = 0.0;
    for (size_t i = 0; i < a.pixels.size(); ++i) {
        const float ch[3] = {std::fabs(a.pixels[i].r - b.pixels[i].r),
                             std::fabs(a.pixels[i].g - b.pixels[i].g),
                             std::fabs(a.pixels[i].b - b.pixels[i].b)};
        for (float c : ch) {
            sum += c;
            d.max_abs = std::max(d.max_abs, static_cast<double>(c));
        }
        d.diff.pixels[i] = {std::fmin(std::fmax(scale * ch[0], 0.0f), 1.0f),
                            std::fmin(std::fmax(scale * ch[1], 0.0f), 1.0f),
                            std::fmin(std::fmax(scale * ch[2], 0.0f), 1.0f)};
    }
    d.mean_abs = a.pixels.empty() ? 0.0 : sum / (3.0 * static_cast<double>(a.pixels.size()));
    return d;
}

std::string stats_to_json(const RenderStats& s, const FrameBuffers& f) {
    std::ostringstream o;
    o.precision(17);
    o << "{\"wall_time_s\": " << s.wall_time_s << ", \"hits\": " << s.hits
      << ", \"lookups\": " << s.lookups << ", \"hit_rate\": " << s.hit_rate
      << ", \"inserts_won\": " << s.inserts_won << ", \"inserts_lost_full\": " << s.inserts_lost_full
      << ", \"width\": " << f.width << ", \"height\": " << f.height << ", \"per_pixel_nodes_found\": [";
    const std::vector<float> avg = f.nodes_found_avg();
    for (size_t i = 0; i < avg.size(); ++i) o << (i ? ", " : "") << avg[i];
    o << "]}";
    return o.str();
}

StatsFile parse_stats_json(std::string_view text) {
    auto number_after = [&](const std::string& key) -> double {
        const size_t k = text.find("\"" + key + "\"");
        if (k == std::string_view::npos) throw std::invalid_argument("stats JSON lacks " + key);
        const size_t c = text.find(':', k);
        return std::stod(std::string(text.substr(c + 1, 32)));
    };
    StatsFile out;
    out.width = static_cast<int>(number_after("width"));
    out.height = static_cast<int>(number_after("height"));
    const size_t k = text.find("\"per_pixel_nodes_found\"");
    if (k == std::string_view::npos) throw std::invalid_argument("stats JSON lacks per_pixel_nodes_found");
    size_t i = text.find('[', k) + 1;
    const size_t end = text.find(']', i);
    while (i < end) {
        const size_t comma = std::min(text.find(',', i), end);
        const std::string tok(text.substr(i, comma - i));
        if (tok.find_first_not_of(" \t\n") != std::string::npos) out.per_pixel_nodes_found.push_back(std::stof(tok));
        i = comma + 1;
    }
    if (out.per_pixel_nodes_found.size() != static_cast<size_t>(out.width) * out.height) {
        throw std::invalid_argument("per_pixel_nodes_found size does not match width*height");
    }
    return out;
}

}  // namespace matcache

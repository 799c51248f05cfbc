// Scene loading and preparation (host side of libmcg), plus the host-only C
// ABI entry points (hashes, codec, audit, scene queries).
//
//   mcg_scene_load   load_scene            src/scene.cpp:300-387
//   build_bvh        Scene::prepare/build  src/scene.cpp:98-194
//   read_ppm_texture read_ppm              src/image.cpp:102-126
//   mcg_hash_*       hash_cell/hash_check  src/cache.cpp:21-39
//   mcg_encode/decode_value                src/cache.cpp:41-71
//   mcg_audit_dump   audit_dump            src/cache.cpp:175-230
//   mcg_camera_setup camera basis + cone_for_camera (src/raycone.cpp:8-13)
//
// The BVH must be the reference's tree node-for-node: closest-hit ties at
// equal t resolve by visit order. It is rebuilt with the same median split
// and the same std::nth_element call over the same primitive order.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cctype>
#include <cmath>
#include <cstring>
#include <fstream>
#include <map>
#include <sstream>
#include <thread>
#include <unordered_map>
#include <unordered_set>

#include <nlohmann/json.hpp>

#include "host_internal.hpp"
#include "host_scene.hpp"

namespace mcg {

namespace {
thread_local std::string g_last_error;
}

void set_last_error(const std::string& msg) { g_last_error = msg; }
void clear_last_error() { g_last_error.clear(); }

using nlohmann::json;

namespace {

[[noreturn]] void scene_error(const std::string& m) { fail(MCG_ERR_SCENE, m); }
[[noreturn]] void image_error(const std::string& m) { fail(MCG_ERR_IMAGE_IO, m); }

std::string slurp(const std::string& path, mcg_status code, const std::string& what) {
    std::ifstream in(path, std::ios::binary);
    if (!in) fail(code, "cannot open " + what + ": " + path);
    std::stringstream ss;
    ss << in.rdbuf();
    return ss.str();
}

std::string parent_dir(const std::string& path) {
    const size_t slash = path.find_last_of('/');
    return slash == std::string::npos ? std::string() : path.substr(0, slash);
}

std::string join_path(const std::string& dir, const std::string& rel) {
    if (dir.empty() || (!rel.empty() && rel[0] == '/')) return rel;
    return dir + "/" + rel;
}

void vec3(const json& j, float out[3]) {
    if (!j.is_array() || j.size() != 3) scene_error("expected a 3-element array");
    for (int k = 0; k < 3; ++k) out[k] = j[k].get<float>();
}

// PPM header token reader: whitespace and '#' comments are skipped; the
// character that ends a token is consumed (image.cpp:21-38).
std::string ppm_token(std::istream& in) {
    std::string tok;
    int c = in.get();
    for (;;) {
        if (c == EOF) break;
        if (c == '#') {
            while (c != EOF && c != '\n') c = in.get();
        } else if (std::isspace(c)) {
            c = in.get();
        } else {
            break;
        }
    }
    while (c != EOF && !std::isspace(c)) {
        tok.push_back(static_cast<char>(c));
        c = in.get();
    }
    return tok;
}

int to_int(const std::string& s, const std::string& path) {
    try {
        return std::stoi(s);
    } catch (const std::exception&) {
        image_error("malformed PPM header: " + path);
    }
}

// ---- geometry helpers with the reference's exact operation order ----------
struct V3 {
    float x, y, z;
};
inline V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V3 add(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3 scale(V3 a, float s) { return {a.x * s, a.y * s, a.z * s}; }
inline float dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline V3 cross(V3 a, V3 b) {
    return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
inline V3 normalize(V3 a) {
    const float len = std::sqrt(dot(a, a));
    return len > 0.0f ? scale(a, 1.0f / len) : V3{0, 0, 0};
}
inline V3 load3(const float* p) { return {p[0], p[1], p[2]}; }

struct Box {
    V3 lo{1e30f, 1e30f, 1e30f};
    V3 hi{-1e30f, -1e30f, -1e30f};
    void grow(V3 p) {
        lo = {std::fmin(lo.x, p.x), std::fmin(lo.y, p.y), std::fmin(lo.z, p.z)};
        hi = {std::fmax(hi.x, p.x), std::fmax(hi.y, p.y), std::fmax(hi.z, p.z)};
    }
    void grow(const Box& b) {
        grow(b.lo);
        grow(b.hi);
    }
    V3 center() const { return scale(add(lo, hi), 0.5f); }
};

}  // namespace

HostTexture read_ppm_texture(const std::string& path, const std::string& ref) {
    std::ifstream in(path, std::ios::binary);
    if (!in) image_error("cannot open: " + path);
    if (ppm_token(in) != "P6") image_error("not a binary PPM file: " + path);
    const int w = to_int(ppm_token(in), path);
    const int h = to_int(ppm_token(in), path);
    const int maxval = to_int(ppm_token(in), path);
    if (w <= 0 || h <= 0 || w > (1 << 16) || h > (1 << 16)) {
        image_error("image dimensions out of range: " + std::to_string(w) + "x" +
                    std::to_string(h));
    }
    if (maxval != 255) image_error("unsupported PPM maxval: " + std::to_string(maxval));
    HostTexture t;
    t.ref = ref;
    t.width = w;
    t.height = h;
    t.rgba.assign(static_cast<size_t>(w) * h * 4, 0.0f);
    std::vector<unsigned char> row(static_cast<size_t>(w) * 3);
    for (int y = 0; y < h; ++y) {
        in.read(reinterpret_cast<char*>(row.data()), static_cast<std::streamsize>(row.size()));
        if (!in) image_error("short read: " + path);
        float* dst = &t.rgba[static_cast<size_t>(y) * w * 4];
        for (int x = 0; x < w; ++x) {
            for (int k = 0; k < 3; ++k) dst[x * 4 + k] = row[x * 3 + k] / 255.0f;
        }
    }
    return t;
}

// ---------------------------------------------------------------------------
// Scene preparation: primitive list, BVH, flat device layout.
// ---------------------------------------------------------------------------
namespace {

struct Prim {
    uint32_t mesh;    // ~0u: sphere
    uint32_t first;   // first index of the triangle
    uint32_t sphere;
};

// The reference's recursive median split (scene.cpp:154-194), producing the
// identical tree faster: primitive boxes and centroids are computed once
// (the reference recomputes them inside every comparison; the values, hence
// every comparison and std::nth_element's permutation, are the same), and
// the top levels build their two subtrees on two threads into private node
// arrays that are then appended in the reference's preorder (node, left
// subtree, right subtree) with child indices rebased.
class BvhBuilder {
public:
    BvhBuilder(const SceneData& s, const std::vector<Prim>& prims, std::vector<uint32_t>& order)
        : order_(order), boxes_(prims.size()), key_{std::vector<float>(prims.size()),
                                                   std::vector<float>(prims.size()),
                                                   std::vector<float>(prims.size())} {
        for (size_t i = 0; i < prims.size(); ++i) {
            Box b;
            const Prim& p = prims[i];
            if (p.mesh != ~0u) {
                const MeshData& m = s.meshes[p.mesh];
                for (int k = 0; k < 3; ++k) b.grow(load3(&m.positions[3 * m.indices[p.first + k]]));
            } else {
                const mcg_sphere_in& sp = s.spheres[p.sphere];
                const V3 c = load3(sp.center);
                const V3 r{sp.radius, sp.radius, sp.radius};
                b.grow(sub(c, r));
                b.grow(add(c, r));
            }
            boxes_[i] = b;
            const V3 c = b.center();
            key_[0][i] = c.x;
            key_[1][i] = c.y;
            key_[2][i] = c.z;
        }
    }

    void run(std::vector<mcg_bvh_node>& nodes) {
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        int depth = 0;
        while ((2u << depth) <= hw && depth < 6) ++depth;  // 2^depth parallel subtrees
        build(0, static_cast<uint32_t>(order_.size()), nodes, order_.size() >= 65536 ? depth : 0);
    }

private:
    // Appends the subtree over order_[first, first+count) to `out`; returns
    // its root's index in `out`.
    int32_t build(uint32_t first, uint32_t count, std::vector<mcg_bvh_node>& out, int par) {
        Box all, centers;
        for (uint32_t i = first; i < first + count; ++i) {
            const Box& b = boxes_[order_[i]];
            all.grow(b);
            centers.grow(b.center());
        }
        const int32_t index = static_cast<int32_t>(out.size());
        out.push_back(mcg_bvh_node{{all.lo.x, all.lo.y, all.lo.z}, 0,
                                   {all.hi.x, all.hi.y, all.hi.z}, 0});
        if (count <= 4) {
            out[index].a = ~static_cast<int32_t>(first);
            out[index].b = static_cast<int32_t>(count);
            return index;
        }
        const V3 ext = sub(centers.hi, centers.lo);
        int axis = 0;
        if (ext.y > ext.x) axis = 1;
        if (ext.z > (axis == 0 ? ext.x : ext.y)) axis = 2;
        const float* key = key_[axis].data();
        const uint32_t mid = first + count / 2;
        std::nth_element(order_.begin() + first, order_.begin() + mid,
                         order_.begin() + first + count,
                         [key](uint32_t a, uint32_t b) { return key[a] < key[b]; });
        if (par <= 0) {
            const int32_t left = build(first, mid - first, out, 0);
            const int32_t right = build(mid, first + count - mid, out, 0);
            out[index].a = left;
            out[index].b = right;
            return index;
        }
        std::vector<mcg_bvh_node> lo, hi;
        std::thread t([&] { build(first, mid - first, lo, par - 1); });
        build(mid, first + count - mid, hi, par - 1);
        t.join();
        const int32_t base_lo = static_cast<int32_t>(out.size());
        append(out, lo, base_lo);
        const int32_t base_hi = static_cast<int32_t>(out.size());
        append(out, hi, base_hi);
        out[index].a = base_lo;
        out[index].b = base_hi;
        return index;
    }

    static void append(std::vector<mcg_bvh_node>& out, const std::vector<mcg_bvh_node>& part,
                       int32_t base) {
        for (mcg_bvh_node n : part) {
            if (n.a >= 0) {  // inner node: a, b are child indices in `part`
                n.a += base;
                n.b += base;
            }
            out.push_back(n);
        }
    }

    std::vector<uint32_t>& order_;
    std::vector<Box> boxes_;
    std::vector<float> key_[3];
};

}  // namespace

void prepare_scene(SceneData& s) {
    std::unordered_map<uint32_t, uint32_t> slot_of;
    for (uint32_t i = 0; i < s.programs.size(); ++i) slot_of[s.programs[i].material_id] = i;
    auto slot = [&](uint32_t material_id) {
        const auto it = slot_of.find(material_id);
        if (it == slot_of.end()) {
            scene_error("material id " + std::to_string(material_id) +
                        " does not resolve to a loaded material");
        }
        return it->second;
    };

    std::vector<Prim> prims;
    std::vector<uint32_t> prim_slot;
    for (uint32_t m = 0; m < s.meshes.size(); ++m) {
        const MeshData& mesh = s.meshes[m];
        if (mesh.positions.size() / 3 != mesh.uvs.size() / 2) {
            scene_error("mesh must carry one uv per vertex");
        }
        if (mesh.indices.size() % 3 != 0) scene_error("mesh indices must be triples");
        const uint32_t nv = static_cast<uint32_t>(mesh.positions.size() / 3);
        for (uint32_t idx : mesh.indices) {
            if (idx >= nv) scene_error("mesh index out of range: " + std::to_string(idx));
        }
        const uint32_t sl = slot(mesh.material_id);
        for (uint32_t i = 0; i < mesh.indices.size(); i += 3) {
            prims.push_back({m, i, 0});
            prim_slot.push_back(sl);
        }
        if (mesh.indices.empty()) (void)sl;
    }
    for (uint32_t k = 0; k < s.spheres.size(); ++k) {
        const uint32_t sl = slot(s.spheres[k].material_id);
        prims.push_back({~0u, 0, k});
        prim_slot.push_back(sl);
    }

    std::vector<uint32_t> order(prims.size());
    for (uint32_t i = 0; i < order.size(); ++i) order[i] = i;
    s.nodes.clear();
    if (!prims.empty()) {
        BvhBuilder(s, prims, order).run(s.nodes);
    }

    // Leaf-ordered primitive arrays.
    const size_t n = prims.size();
    s.prim_geom.assign(n * 12, 0.0f);
    s.prim_uv.assign(n * 6, 0.0f);
    s.prim_info.assign(n, 0);
    s.prim_source.assign(n, 0);
    for (size_t i = 0; i < n; ++i) {
        const Prim& p = prims[order[i]];
        float* g = &s.prim_geom[i * 12];
        s.prim_source[i] = order[i];
        if (p.mesh != ~0u) {
            const MeshData& m = s.meshes[p.mesh];
            const uint32_t i0 = m.indices[p.first], i1 = m.indices[p.first + 1],
                           i2 = m.indices[p.first + 2];
            const V3 p0 = load3(&m.positions[3 * i0]);
            const V3 e1 = sub(load3(&m.positions[3 * i1]), p0);
            const V3 e2 = sub(load3(&m.positions[3 * i2]), p0);
            const float vals[12] = {p0.x, p0.y, p0.z, 0, e1.x, e1.y, e1.z, 0, e2.x, e2.y, e2.z, 0};
            std::memcpy(g, vals, sizeof(vals));
            float* uv = &s.prim_uv[i * 6];
            uv[0] = m.uvs[2 * i0]; uv[1] = m.uvs[2 * i0 + 1];
            uv[2] = m.uvs[2 * i1]; uv[3] = m.uvs[2 * i1 + 1];
            uv[4] = m.uvs[2 * i2]; uv[5] = m.uvs[2 * i2 + 1];
            s.prim_info[i] = prim_slot[order[i]];
        } else {
            const mcg_sphere_in& sp = s.spheres[p.sphere];
            g[0] = sp.center[0]; g[1] = sp.center[1]; g[2] = sp.center[2]; g[3] = sp.radius;
            s.prim_info[i] = prim_slot[order[i]] | MCG_PRIM_SPHERE;
        }
    }
}

void flatten_programs(SceneData& s) {
    s.code.clear(); s.consts.clear(); s.noise.clear(); s.ramps.clear(); s.ramp_stops.clear();
    s.flat_programs.clear();
    for (const Program& p : s.programs) {
        mcg_program fp{};
        fp.material_id = p.material_id;
        fp.code_offset = static_cast<uint32_t>(s.code.size());
        fp.code_len = static_cast<uint32_t>(p.code.size());
        fp.max_stack = static_cast<uint32_t>(p.max_stack);
        fp.cache_point_count = p.cache_point_count;
        const uint32_t cbase = static_cast<uint32_t>(s.consts.size());
        const uint32_t nbase = static_cast<uint32_t>(s.noise.size());
        const uint32_t rbase = static_cast<uint32_t>(s.ramps.size());
        for (mcg_insn ins : p.code) {
            if (ins.op == MCG_OP_PUSH_CONST) ins.arg += cbase;
            if (ins.op == MCG_OP_NOISE) ins.arg += nbase;
            if (ins.op == MCG_OP_RAMP) ins.arg += rbase;
            s.code.push_back(ins);
        }
        s.consts.insert(s.consts.end(), p.consts.begin(), p.consts.end());
        s.noise.insert(s.noise.end(), p.noise.begin(), p.noise.end());
        for (const auto& stops : p.ramps) {
            s.ramps.push_back({static_cast<uint32_t>(s.ramp_stops.size()),
                               static_cast<uint32_t>(stops.size())});
            s.ramp_stops.insert(s.ramp_stops.end(), stops.begin(), stops.end());
        }
        s.flat_programs.push_back(fp);
    }
    s.tex_table.clear();
    s.texels.clear();
    for (const HostTexture& t : s.textures) {
        s.tex_table.push_back({t.width, t.height, static_cast<uint64_t>(s.texels.size() / 4)});
        s.texels.insert(s.texels.end(), t.rgba.begin(), t.rgba.end());
    }
}

void fill_flat(const SceneData& s, mcg_flat_scene* f) {
    std::memset(f, 0, sizeof(*f));
    std::memcpy(f->cam_position, s.cam_position, sizeof(f->cam_position));
    std::memcpy(f->cam_look_at, s.cam_look_at, sizeof(f->cam_look_at));
    std::memcpy(f->cam_up, s.cam_up, sizeof(f->cam_up));
    f->cam_vfov_deg = s.cam_vfov_deg;
    f->cam_width = s.cam_width;
    f->cam_height = s.cam_height;
    std::memcpy(f->env, s.env, sizeof(f->env));
    f->n_prims = static_cast<uint32_t>(s.prim_info.size());
    f->prim_geom = s.prim_geom.data();
    f->prim_uv = s.prim_uv.data();
    f->prim_info = s.prim_info.data();
    f->n_nodes = static_cast<uint32_t>(s.nodes.size());
    f->nodes = s.nodes.data();
    f->n_point_lights = static_cast<uint32_t>(s.point_lights.size());
    f->point_lights = s.point_lights.data();
    f->n_rect_lights = static_cast<uint32_t>(s.rect_lights.size());
    f->rect_lights = s.rect_lights.data();
    f->n_programs = static_cast<uint32_t>(s.flat_programs.size());
    f->programs = s.flat_programs.data();
    f->n_code = static_cast<uint32_t>(s.code.size());
    f->code = s.code.data();
    f->n_consts = static_cast<uint32_t>(s.consts.size());
    f->consts = s.consts.data();
    f->n_noise = static_cast<uint32_t>(s.noise.size());
    f->noise = s.noise.data();
    f->n_ramps = static_cast<uint32_t>(s.ramps.size());
    f->ramps = s.ramps.data();
    f->n_ramp_stops = static_cast<uint32_t>(s.ramp_stops.size());
    f->ramp_stops = s.ramp_stops.data();
    f->n_textures = static_cast<uint32_t>(s.tex_table.size());
    f->textures = s.tex_table.data();
    f->n_texels = s.texels.size() / 4;
    f->texels = s.texels.data();
}

// MCG_LOAD_TIMING=1: per-phase wall times of a scene load on stderr.
struct LoadTimer {
    bool on = std::getenv("MCG_LOAD_TIMING") != nullptr;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void phase(const char* name) {
        if (!on) return;
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[mcg load] %-20s %8.3f s\n", name,
                     std::chrono::duration<double>(now - t).count());
        t = now;
    }
};

SceneData load_scene_file(const std::string& path, int min_subtree_size) {
    LoadTimer timer;
    const std::string text = slurp(path, MCG_ERR_SCENE, "scene file");
    timer.phase("read");
    json doc;
    try {
        doc = json::parse(text);
        timer.phase("json parse");
    } catch (const json::parse_error& e) {
        scene_error(std::string("scene JSON parse error: ") + e.what());
    }
    SceneData s;
    const std::string dir = parent_dir(path);
    try {
        const json& cam = doc.at("camera");
        vec3(cam.at("position"), s.cam_position);
        vec3(cam.at("look_at"), s.cam_look_at);
        if (cam.contains("up")) vec3(cam.at("up"), s.cam_up);
        s.cam_vfov_deg = cam.at("vfov_deg").get<float>();
        s.cam_width = cam.value("width", 256);
        s.cam_height = cam.value("height", 256);

        for (const auto& jm : doc.value("materials", json::array())) {
            const std::string file = join_path(dir, jm.get<std::string>());
            const Graph g = parse_graph(slurp(file, MCG_ERR_GRAPH, "material file"));
            // Textures resolve relative to the material file; the pool is
            // keyed by reference string (texture.cpp:56-67).
            for (const GNode& n : g.nodes) {
                if (n.kind != Kind::TexImage) continue;
                bool have = false;
                for (const HostTexture& t : s.textures) have = have || t.ref == n.image;
                if (!have) {
                    s.textures.push_back(read_ppm_texture(join_path(parent_dir(file), n.image),
                                                          n.image));
                }
            }
            std::vector<std::string> refs;
            for (const HostTexture& t : s.textures) refs.push_back(t.ref);
            s.analyses.push_back(analyze_graph(g, min_subtree_size));
            s.programs.push_back(compile_analysis(s.analyses.back(), refs));
        }
        for (const auto& jm : doc.value("meshes", json::array())) {
            MeshData m;
            const auto& pos = jm.at("positions");
            for (size_t i = 0; i + 2 < pos.size(); i += 3) {
                for (int k = 0; k < 3; ++k) m.positions.push_back(pos[i + k].get<float>());
            }
            const auto& uvs = jm.at("uvs");
            for (size_t i = 0; i + 1 < uvs.size(); i += 2) {
                m.uvs.push_back(uvs[i].get<float>());
                m.uvs.push_back(uvs[i + 1].get<float>());
            }
            for (const auto& idx : jm.at("indices")) m.indices.push_back(idx.get<uint32_t>());
            m.material_id = jm.at("material").get<uint32_t>();
            s.meshes.push_back(std::move(m));
        }
        for (const auto& js : doc.value("spheres", json::array())) {
            mcg_sphere_in sp{};
            vec3(js.at("center"), sp.center);
            sp.radius = js.at("radius").get<float>();
            sp.material_id = js.at("material").get<uint32_t>();
            s.spheres.push_back(sp);
        }
        for (const auto& jl : doc.value("lights", json::array())) {
            const std::string type = jl.at("type").get<std::string>();
            if (type == "point") {
                mcg_point_light l{};
                vec3(jl.at("position"), l.position);
                vec3(jl.at("intensity"), l.intensity);
                s.point_lights.push_back(l);
            } else if (type == "rect") {
                mcg_rect_light l{};
                vec3(jl.at("corner"), l.corner);
                vec3(jl.at("edge_u"), l.edge_u);
                vec3(jl.at("edge_v"), l.edge_v);
                vec3(jl.at("radiance"), l.radiance);
                s.rect_lights.push_back(l);
            } else {
                scene_error("unknown light type '" + type + "'");
            }
        }
        if (doc.contains("env")) vec3(doc.at("env"), s.env);
    } catch (const json::exception& e) {
        scene_error(std::string("scene JSON schema error: ") + e.what());
    }
    timer.phase("materials + meshes");
    flatten_programs(s);
    prepare_scene(s);
    timer.phase("bvh + flat layout");
    return s;
}

// Camera basis and primary cone. The pinned tracer:
// forward = normalize(look_at - position), right = normalize(cross(forward,
// up)), up' = cross(right, forward); tan_half = tanf(vfov/2); spread per
// cone_for_camera with the render height.
void camera_setup(const mcg_flat_scene& f, int32_t w, int32_t h, float out[12]) {
    const V3 pos = load3(f.cam_position);
    const V3 fwd = normalize(sub(load3(f.cam_look_at), pos));
    const V3 right = normalize(cross(fwd, load3(f.cam_up)));
    const V3 up = cross(right, fwd);
    const float vfov = f.cam_vfov_deg * (3.14159265358979323846f / 180.0f);
    const float tan_half = std::tan(vfov * 0.5f);
    const float spread = std::atan(2.0f * std::tan(vfov * 0.5f) / static_cast<float>(h));
    const float vals[12] = {fwd.x, fwd.y, fwd.z, right.x, right.y, right.z, up.x, up.y, up.z,
                            tan_half, static_cast<float>(w) / static_cast<float>(h), spread};
    std::memcpy(out, vals, sizeof(vals));
}

}  // namespace mcg

// ===========================================================================
// Host-only C ABI
// ===========================================================================
using namespace mcg;

struct mcg_scene {
    SceneData data;
};

extern "C" {

const char* mcg_last_error(void) { return g_last_error.c_str(); }
int mcg_abi_version(void) { return MCG_ABI_VERSION; }

static inline uint64_t splitmix_fin(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

static uint64_t descriptor_chain(const mcg_descriptor* d, uint64_t h) {
    h = splitmix_fin(h ^ (static_cast<uint64_t>(d->mat_idx) | (static_cast<uint64_t>(d->node_idx) << 32)));
    h = splitmix_fin(h ^ (static_cast<uint64_t>(d->texel_x) | (static_cast<uint64_t>(d->texel_y) << 32)));
    return splitmix_fin(h ^ static_cast<uint64_t>(d->mip_level));
}

uint64_t mcg_hash_cell(const mcg_descriptor* d) { return descriptor_chain(d, 0x243f6a8885a308d3ull); }

uint32_t mcg_hash_check(const mcg_descriptor* d) {
    const uint32_t h = static_cast<uint32_t>(descriptor_chain(d, 0x13198a2e03707344ull));
    return h ? h : 1u;
}

uint32_t mcg_encode_value(const float rgb[3]) {
    double c[3];
    for (int k = 0; k < 3; ++k) c[k] = (std::isfinite(rgb[k]) && rgb[k] > 0.0f) ? rgb[k] : 0.0;
    const double m = std::fmax(c[0], std::fmax(c[1], c[2]));
    if (m <= 0.0) return 0;
    int e = 0;
    std::frexp(m, &e);
    if (e < -127) return 0;
    if (e > 127) e = 127;
    const double f = std::ldexp(256.0, -e);
    uint32_t word = static_cast<uint32_t>(e + 128) << 24;
    for (int k = 0; k < 3; ++k) {
        const uint32_t q = static_cast<uint32_t>(c[k] * f);
        word |= (q > 255 ? 255u : q) << (16 - 8 * k);
    }
    return word;
}

void mcg_decode_value(uint32_t packed, float rgb_out[3]) {
    const uint32_t e = packed >> 24;
    if (e == 0) {
        rgb_out[0] = rgb_out[1] = rgb_out[2] = 0.0f;
        return;
    }
    const double s = std::ldexp(1.0, static_cast<int>(e) - 136);
    for (int k = 0; k < 3; ++k) {
        rgb_out[k] = static_cast<float>((((packed >> (16 - 8 * k)) & 255u) + 0.5) * s);
    }
}

mcg_status mcg_memory_bytes(uint64_t n_cells, uint64_t n_entries, uint64_t* bytes_out) {
    return guarded([&] {
        uint64_t bytes = 0;
        if (n_cells != 0 && n_entries != 0) {
            const uint64_t slots = n_cells * n_entries;
            if (slots / n_entries != n_cells || slots > UINT64_MAX / 8) {
                fail(MCG_ERR_OVERFLOW, "cache size overflows 64 bits");
            }
            bytes = slots * 8;
        }
        if (bytes_out) *bytes_out = bytes;
    });
}

mcg_status mcg_audit_dump(const char* path, mcg_audit_report* out) {
    return guarded([&] {
        if (!path || !out) fail(MCG_ERR_INVALID_ARGUMENT, "null argument");
        std::memset(out, 0, sizeof(*out));
        out->bad_cell = -1;
        auto problem = [&](const std::string& m) {
            std::snprintf(out->problem, sizeof(out->problem), "%s", m.c_str());
        };
        std::ifstream in(path, std::ios::binary);
        if (!in) return problem(std::string("cannot open dump: ") + path);
        uint64_t header[2] = {0, 0};
        in.read(reinterpret_cast<char*>(header), sizeof(header));
        if (!in) return problem("truncated header");
        out->n_cells = header[0];
        out->n_entries = header[1];
        if (header[0] == 0 || header[1] == 0 || header[1] > (1u << 20)) {
            return problem("implausible table dimensions");
        }
        std::vector<uint64_t> cell(header[1]);
        std::unordered_set<uint32_t> seen;
        for (uint64_t c = 0; c < header[0]; ++c) {
            in.read(reinterpret_cast<char*>(cell.data()),
                    static_cast<std::streamsize>(cell.size() * 8));
            if (!in) return problem("truncated at cell " + std::to_string(c));
            seen.clear();
            for (uint64_t w : cell) {
                if (w == 0) continue;
                ++out->occupied;
                const uint32_t h = static_cast<uint32_t>(w >> 32);
                if (h == 0) {
                    out->bad_cell = static_cast<int64_t>(c);
                    return problem("occupied slot with zero check-hash in cell " +
                                   std::to_string(c));
                }
                if (!seen.insert(h).second) {
                    out->bad_cell = static_cast<int64_t>(c);
                    return problem("duplicate check-hash in cell " + std::to_string(c));
                }
            }
        }
        in.peek();
        if (!in.eof()) return problem("trailing bytes after table");
        out->clean = 1;
    });
}

mcg_status mcg_scene_load(const char* path, int32_t min_subtree_size, mcg_scene** out) {
    return guarded([&] {
        if (!path || !out) fail(MCG_ERR_INVALID_ARGUMENT, "null argument");
        auto* s = new mcg_scene;
        try {
            s->data = load_scene_file(path, min_subtree_size);
        } catch (...) {
            delete s;
            throw;
        }
        *out = s;
    });
}

mcg_status mcg_scene_build(const mcg_scene_in* in, mcg_scene** out) {
    return guarded([&] {
        if (!in || !out) fail(MCG_ERR_INVALID_ARGUMENT, "null argument");
        auto* s = new mcg_scene;
        try {
            SceneData& d = s->data;
            std::memcpy(d.cam_position, in->cam_position, sizeof(d.cam_position));
            std::memcpy(d.cam_look_at, in->cam_look_at, sizeof(d.cam_look_at));
            std::memcpy(d.cam_up, in->cam_up, sizeof(d.cam_up));
            d.cam_vfov_deg = in->cam_vfov_deg;
            d.cam_width = in->cam_width;
            d.cam_height = in->cam_height;
            std::memcpy(d.env, in->env, sizeof(d.env));
            for (uint32_t i = 0; i < in->n_meshes; ++i) {
                const mcg_mesh_in& mi = in->meshes[i];
                MeshData m;
                m.positions.assign(mi.positions, mi.positions + 3 * mi.n_vertices);
                m.uvs.assign(mi.uvs, mi.uvs + 2 * mi.n_vertices);
                m.indices.assign(mi.indices, mi.indices + mi.n_indices);
                m.material_id = mi.material_id;
                d.meshes.push_back(std::move(m));
            }
            d.spheres.assign(in->spheres, in->spheres + in->n_spheres);
            d.point_lights.assign(in->point_lights, in->point_lights + in->n_point_lights);
            d.rect_lights.assign(in->rect_lights, in->rect_lights + in->n_rect_lights);
            // Programs arrive flattened: keep them as they are.
            for (uint32_t i = 0; i < in->n_programs; ++i) {
                Program p;
                p.material_id = in->programs[i].material_id;
                d.programs.push_back(p);
            }
            d.flat_programs.assign(in->programs, in->programs + in->n_programs);
            d.code.assign(in->code, in->code + in->n_code);
            d.consts.assign(in->consts, in->consts + in->n_consts);
            d.noise.assign(in->noise, in->noise + in->n_noise);
            d.ramps.assign(in->ramps, in->ramps + in->n_ramps);
            d.ramp_stops.assign(in->ramp_stops, in->ramp_stops + in->n_ramp_stops);
            d.tex_table.assign(in->textures, in->textures + in->n_textures);
            d.texels.assign(in->texels, in->texels + 4 * in->n_texels);
            prepare_scene(d);
        } catch (...) {
            delete s;
            throw;
        }
        *out = s;
    });
}

mcg_status mcg_schedule_program(mcg_insn* code, uint32_t n_code, const mcg_const* consts,
                                uint32_t n_consts, uint32_t* max_stack) {
    return guarded([&] {
        if (!code || n_code == 0 || (!consts && n_consts)) fail(MCG_ERR_INVALID_ARGUMENT, "null argument");
        Program p;
        p.code.assign(code, code + n_code);
        p.consts.assign(consts, consts + n_consts);
        if (p.code.back().op != MCG_OP_END) fail(MCG_ERR_COMPILE, "program must end with End");
        int depth = 0, peak = 0;
        for (const mcg_insn& ins : p.code) {
            if (ins.op > MCG_OP_END) fail(MCG_ERR_COMPILE, "unknown opcode");
            if (ins.op == MCG_OP_PUSH_CONST && ins.arg >= n_consts) {
                fail(MCG_ERR_COMPILE, "constant index out of range");
            }
            if (ins.op == MCG_OP_END) break;
            switch (ins.op) {
                case MCG_OP_ADD: case MCG_OP_SUB: case MCG_OP_MUL: case MCG_OP_DIV:
                case MCG_OP_DOT: case MCG_OP_POWER: depth -= 1; break;
                case MCG_OP_MIX: depth -= 2; break;
                case MCG_OP_PUSH_CONST: case MCG_OP_LOAD_UV: case MCG_OP_LOAD_POSITION:
                case MCG_OP_LOAD_NORMAL: case MCG_OP_LOAD_INCOMING: case MCG_OP_TEX_SAMPLE:
                case MCG_OP_CHECKER: case MCG_OP_NOISE: depth += 1; break;
                default: break;
            }
            if (depth <= 0) fail(MCG_ERR_COMPILE, "stack underflow during compilation");
            peak = std::max(peak, depth);
        }
        if (depth != 1) fail(MCG_ERR_COMPILE, "unbalanced stack effect: final depth " + std::to_string(depth));
        if (peak > 255) fail(MCG_ERR_COMPILE, "stack depth exceeds 255");
        schedule_program(p);
        std::copy(p.code.begin(), p.code.end(), code);
        if (max_stack) *max_stack = static_cast<uint32_t>(peak);
    });
}

mcg_status mcg_scene_destroy(mcg_scene* scene) {
    delete scene;
    return MCG_OK;
}

mcg_status mcg_scene_flat(const mcg_scene* scene, mcg_flat_scene* out) {
    return guarded([&] {
        if (!scene || !out) fail(MCG_ERR_INVALID_ARGUMENT, "null argument");
        fill_flat(scene->data, out);
    });
}

static mcg_status copy_text(const std::string& text, char* buf, size_t cap, size_t* len_out) {
    if (len_out) *len_out = text.size();
    if (buf && cap > 0) {
        const size_t n = std::min(cap - 1, text.size());
        std::memcpy(buf, text.data(), n);
        buf[n] = '\0';
    }
    return MCG_OK;
}

mcg_status mcg_scene_disassemble(const mcg_scene* scene, uint32_t slot, char* buf, size_t cap,
                                 size_t* len_out) {
    return guarded([&] {
        if (!scene || slot >= scene->data.programs.size() || scene->data.analyses.empty()) {
            fail(MCG_ERR_INVALID_ARGUMENT, "no compiled program at that slot");
        }
        copy_text(disassemble_program(scene->data.programs[slot]), buf, cap, len_out);
    });
}

mcg_status mcg_scene_analysis_json(const mcg_scene* scene, uint32_t slot, char* buf, size_t cap,
                                   size_t* len_out) {
    return guarded([&] {
        if (!scene || slot >= scene->data.analyses.size()) {
            fail(MCG_ERR_INVALID_ARGUMENT, "no analysis at that slot");
        }
        copy_text(analysis_json(scene->data.analyses[slot]), buf, cap, len_out);
    });
}

mcg_status mcg_camera_setup(const mcg_flat_scene* scene, int32_t width, int32_t height,
                            float out[12]) {
    return guarded([&] {
        if (!scene || !out || width <= 0 || height <= 0) {
            fail(MCG_ERR_INVALID_ARGUMENT, "invalid camera set-up arguments");
        }
        camera_setup(*scene, width, height, out);
    });
}

}  // extern "C"

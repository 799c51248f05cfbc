// Material graphs -> analysis -> device bytecode (host side of libmcg).
//
// Behavioural contract (paths relative to /root/reference/proj/core):
//   parse_graph      load_graph + parse_params      src/graph.cpp:88-287
//   check_graph      validate_graph                 src/graph.cpp:297-333
//   analyze_graph    fold/classify/select/uses_uv   src/analysis.cpp:73-156
//   compile_analysis Emitter + compile              src/stackvm.cpp:15-246
//   schedule_program (new) static stack slots/tags for the warp-uniform VM
//   disassemble_program  disassemble                src/stackvm.cpp:370-443
//
// Constant folding evaluates through the host's libm (sinf/powf) exactly as
// the reference's apply_math_node does (src/eval.cpp:7-24, include/value.hpp),
// so folded constants are bit-identical to the reference's.
#include <algorithm>
#include <cmath>
#include <map>
#include <sstream>

#include <nlohmann/json.hpp>

#include "host_internal.hpp"

namespace mcg {

using nlohmann::json;

namespace {

struct KindInfo {
    Kind kind;
    const char* label;
    int arity;
    uint8_t dep;  // intrinsic class (analysis.cpp:11-37): 0 Const, 1 Uv, 2 Other
};

constexpr KindInfo kKinds[] = {
    {Kind::ConstFloat, "const_float", 0, 0}, {Kind::ConstColor, "const_color", 0, 0},
    {Kind::Uv, "uv", 0, 1},                  {Kind::Position, "position", 0, 2},
    {Kind::Normal, "normal", 0, 2},          {Kind::Incoming, "incoming", 0, 2},
    {Kind::TexImage, "tex_image", 0, 1},     {Kind::Checker, "checker", 0, 1},
    {Kind::NoiseFbm, "noise_fbm", 0, 1},     {Kind::Add, "add", 2, 0},
    {Kind::Sub, "sub", 2, 0},                {Kind::Mul, "mul", 2, 0},
    {Kind::Div, "div", 2, 0},                {Kind::Mix, "mix", 3, 0},
    {Kind::Clamp, "clamp", 1, 0},            {Kind::Dot, "dot", 2, 0},
    {Kind::SinWave, "sin_wave", 1, 0},       {Kind::ColorRamp, "color_ramp", 1, 0},
    {Kind::Power, "power", 2, 0},            {Kind::BsdfDiffuse, "bsdf_diffuse", 1, 2},
    {Kind::BsdfOutput, "bsdf_output", 1, 2},
};

const KindInfo& info(Kind k) { return kKinds[static_cast<int>(k)]; }

std::string node_msg(const std::string& m, uint32_t id) {
    return m + " (node " + std::to_string(id) + ")";
}

[[noreturn]] void graph_error(const std::string& m) { fail(MCG_ERR_GRAPH, m); }
[[noreturn]] void graph_error(const std::string& m, uint32_t id) {
    fail(MCG_ERR_GRAPH, node_msg(m, id));
}

void read_rgb(const json& j, uint32_t id, float out[3]) {
    if (!j.is_array() || j.size() != 3) graph_error("rgb parameter must be a 3-element array", id);
    for (int k = 0; k < 3; ++k) out[k] = j[k].get<float>();
    if (!std::isfinite(out[0]) || !std::isfinite(out[1]) || !std::isfinite(out[2])) {
        graph_error("rgb components must be finite", id);
    }
}

// Kind-specific parameter block (graph.cpp:88-166).
void read_params(GNode& n, const json& p, uint32_t id) {
    switch (n.kind) {
        case Kind::ConstFloat: {
            const float v = p.value("value", 0.0f);
            if (!std::isfinite(v)) graph_error("const_float value must be finite", id);
            n.value = HVal::s(v);
            break;
        }
        case Kind::ConstColor: {
            float c[3];
            read_rgb(p.value("rgb", json::array({0.0, 0.0, 0.0})), id, c);
            n.value = HVal::c(c[0], c[1], c[2]);
            break;
        }
        case Kind::Uv: {
            const std::string ch = p.value("channel", "uv");
            if (ch == "uv") n.uv_channel = 0;
            else if (ch == "u") n.uv_channel = 1;
            else if (ch == "v") n.uv_channel = 2;
            else graph_error("unknown uv channel '" + ch + "'", id);
            break;
        }
        case Kind::TexImage: {
            if (!p.contains("image") || !p["image"].is_string()) {
                graph_error("tex_image requires an 'image' reference", id);
            }
            n.image = p["image"].get<std::string>();
            const std::string wrap = p.value("wrap", "repeat");
            if (wrap == "repeat") n.wrap_clamp = false;
            else if (wrap == "clamp") n.wrap_clamp = true;
            else graph_error("unknown wrap mode '" + wrap + "'", id);
            break;
        }
        case Kind::Checker:
            n.checker_scale = p.value("scale", 1.0f);
            if (!std::isfinite(n.checker_scale)) graph_error("checker scale must be finite", id);
            break;
        case Kind::NoiseFbm:
            n.noise.octaves = p.value("octaves", 4);
            n.noise.frequency = p.value("frequency", 1.0f);
            n.noise.lacunarity = p.value("lacunarity", 2.0f);
            n.noise.gain = p.value("gain", 0.5f);
            if (n.noise.octaves < 1 || n.noise.octaves > 10) {
                graph_error("noise_fbm octaves must be in [1, 10]", id);
            }
            if (!std::isfinite(n.noise.frequency) || !std::isfinite(n.noise.lacunarity) ||
                !std::isfinite(n.noise.gain)) {
                graph_error("noise_fbm parameters must be finite", id);
            }
            break;
        case Kind::ColorRamp: {
            if (!p.contains("stops") || !p["stops"].is_array() || p["stops"].empty()) {
                graph_error("color_ramp requires a non-empty 'stops' array", id);
            }
            for (const auto& js : p["stops"]) {
                mcg_ramp_stop st{};
                st.t = js.value("t", 0.0f);
                float c[3];
                read_rgb(js.value("rgb", json::array({0.0, 0.0, 0.0})), id, c);
                st.r = c[0];
                st.g = c[1];
                st.b = c[2];
                if (!std::isfinite(st.t)) graph_error("ramp stop position must be finite", id);
                n.stops.push_back(st);
            }
            for (size_t i = 1; i < n.stops.size(); ++i) {
                if (n.stops[i].t < n.stops[i - 1].t) {
                    graph_error("ramp stops must be sorted by position", id);
                }
            }
            break;
        }
        default:
            break;
    }
}

// ---- value kernels used by constant folding (value.hpp:92-156) -----------

template <typename F>
HVal lanewise2(const HVal& a, const HVal& b, F f) {
    const float r = f(a.x, b.x), g = f(a.y, b.y), bl = f(a.z, b.z);
    return (a.scalar && b.scalar) ? HVal::s(r) : HVal::c(r, g, bl);
}

template <typename F>
HVal lanewise1(const HVal& a, F f) {
    const float r = f(a.x), g = f(a.y), b = f(a.z);
    return a.scalar ? HVal::s(r) : HVal::c(r, g, b);
}

HVal fold_node(const GNode& n, const HVal* v) {
    switch (n.kind) {
        case Kind::Add: return lanewise2(v[0], v[1], [](float x, float y) { return x + y; });
        case Kind::Sub: return lanewise2(v[0], v[1], [](float x, float y) { return x - y; });
        case Kind::Mul: return lanewise2(v[0], v[1], [](float x, float y) { return x * y; });
        case Kind::Div:
            return lanewise2(v[0], v[1], [](float x, float y) { return y == 0.0f ? 0.0f : x / y; });
        case Kind::Mix: {
            const float t = v[2].lum();
            return lanewise2(v[0], v[1], [t](float x, float y) { return x * (1.0f - t) + y * t; });
        }
        case Kind::Clamp:
            return lanewise1(v[0], [](float x) { return std::fmin(std::fmax(x, 0.0f), 1.0f); });
        case Kind::Dot: return HVal::s(v[0].x * v[1].x + v[0].y * v[1].y + v[0].z * v[1].z);
        case Kind::SinWave:
            return lanewise1(v[0], [](float x) {
                return 0.5f + 0.5f * std::sin(x * 6.28318530717958647692f);
            });
        case Kind::Power:
            return lanewise2(v[0], v[1], [](float x, float y) {
                const float r = std::pow(std::fmax(x, 0.0f), y);
                return std::isfinite(r) ? r : 0.0f;
            });
        case Kind::ColorRamp: {
            const auto& s = n.stops;
            const float t = v[0].lum();
            if (t <= s.front().t) return HVal::c(s.front().r, s.front().g, s.front().b);
            if (t >= s.back().t) return HVal::c(s.back().r, s.back().g, s.back().b);
            for (size_t i = 1; i < s.size(); ++i) {
                if (t <= s[i].t) {
                    const float span = s[i].t - s[i - 1].t;
                    const float w = span > 0.0f ? (t - s[i - 1].t) / span : 0.0f;
                    const float u = 1.0f - w;
                    return HVal::c(s[i - 1].r * u + s[i].r * w, s[i - 1].g * u + s[i].g * w,
                                   s[i - 1].b * u + s[i].b * w);
                }
            }
            return HVal::c(s.back().r, s.back().g, s.back().b);
        }
        default:
            graph_error("fold on non-math node");
    }
}

bool is_const(Kind k) { return k == Kind::ConstFloat || k == Kind::ConstColor; }
bool is_math(Kind k) { return info(k).dep == 0 && info(k).arity > 0; }

size_t closure_size(const Graph& g, uint32_t root) {
    std::vector<uint8_t> seen(g.nodes.size(), 0);
    std::vector<uint32_t> work{root};
    seen[root] = 1;
    size_t count = 1;
    while (!work.empty()) {
        const uint32_t n = work.back();
        work.pop_back();
        for (uint32_t in : g.nodes[n].in) {
            if (!seen[in]) {
                seen[in] = 1;
                ++count;
                work.push_back(in);
            }
        }
    }
    return count;
}

}  // namespace

int arity(Kind k) { return info(k).arity; }
const char* kind_label(Kind k) { return info(k).label; }

Graph parse_graph(const std::string& text) {
    json doc;
    try {
        doc = json::parse(text);
    } catch (const json::parse_error& e) {
        graph_error(std::string("material JSON parse error: ") + e.what());
    }
    Graph g;
    try {
        g.material_id = doc.at("material_id").get<uint32_t>();
        g.output = doc.at("output").get<uint32_t>();
        const json& nodes = doc.at("nodes");
        if (!nodes.is_array()) graph_error("'nodes' must be an array");
        g.nodes.reserve(nodes.size());
        for (size_t pos = 0; pos < nodes.size(); ++pos) {
            const json& jn = nodes[pos];
            const uint32_t id = jn.at("id").get<uint32_t>();
            if (id != pos) {
                graph_error("node ids must be dense 0..N-1; found id " + std::to_string(id) +
                                " at position " + std::to_string(pos),
                            id);
            }
            const std::string label = jn.at("kind").get<std::string>();
            const KindInfo* found = nullptr;
            for (const KindInfo& ki : kKinds) {
                if (label == ki.label) found = &ki;
            }
            if (!found) graph_error("unknown node kind '" + label + "'", id);
            GNode n;
            n.kind = found->kind;
            read_params(n, jn.value("params", json::object()), id);
            if (jn.contains("inputs")) {
                for (const auto& in : jn.at("inputs")) n.in.push_back(in.get<uint32_t>());
            }
            g.nodes.push_back(std::move(n));
        }
    } catch (const json::exception& e) {
        graph_error(std::string("material JSON schema error: ") + e.what());
    }
    check_graph(g);
    return g;
}

void check_graph(const Graph& g) {
    if (g.nodes.empty()) graph_error("graph has no nodes");
    size_t outputs = 0;
    for (uint32_t id = 0; id < g.nodes.size(); ++id) {
        const GNode& n = g.nodes[id];
        if (static_cast<int>(n.in.size()) != arity(n.kind)) {
            graph_error("arity mismatch for " + std::string(kind_label(n.kind)) + ": expected " +
                            std::to_string(arity(n.kind)) + " inputs, got " +
                            std::to_string(n.in.size()),
                        id);
        }
        for (uint32_t in : n.in) {
            if (in >= g.nodes.size()) graph_error("dangling input id " + std::to_string(in), id);
            if (in >= id) {
                graph_error("cycle detected: input " + std::to_string(in) +
                                " does not precede its consumer",
                            id);
            }
        }
        outputs += n.kind == Kind::BsdfOutput;
    }
    if (outputs != 1) {
        graph_error("graph must contain exactly one bsdf_output node, found " +
                    std::to_string(outputs));
    }
    if (g.output >= g.nodes.size()) {
        graph_error("output node id out of range: " + std::to_string(g.output));
    }
    if (g.nodes[g.output].kind != Kind::BsdfOutput) {
        graph_error("output node must be the bsdf_output node", g.output);
    }
}

Analysis analyze_graph(const Graph& src, int min_subtree_size) {
    // fold_constants (analysis.cpp:73-109): ids are topological, one forward
    // sweep collapses whole constant chains.
    std::vector<GNode> nodes = src.nodes;
    for (GNode& n : nodes) {
        if (!is_math(n.kind)) continue;
        bool all_const = true;
        for (uint32_t in : n.in) all_const = all_const && is_const(nodes[in].kind);
        if (!all_const) continue;
        HVal args[3];
        for (size_t i = 0; i < n.in.size(); ++i) args[i] = nodes[n.in[i]].value;
        const HVal v = fold_node(n, args);
        GNode c;
        c.kind = v.scalar ? Kind::ConstFloat : Kind::ConstColor;
        c.value = v.scalar ? HVal::s(v.x) : v;
        n = std::move(c);
    }
    std::vector<uint8_t> live(nodes.size(), 0);
    live[src.output] = 1;
    for (uint32_t id = src.output + 1; id-- > 0;) {
        if (!live[id]) continue;
        for (uint32_t in : nodes[id].in) live[in] = 1;
    }
    Analysis a;
    a.remap.assign(nodes.size(), ~uint32_t{0});
    a.graph.material_id = src.material_id;
    for (uint32_t id = 0; id < nodes.size(); ++id) {
        if (!live[id]) continue;
        a.remap[id] = static_cast<uint32_t>(a.graph.nodes.size());
        GNode n = std::move(nodes[id]);
        for (uint32_t& in : n.in) in = a.remap[in];
        a.graph.nodes.push_back(std::move(n));
    }
    a.graph.output = a.remap[src.output];

    // classify_deps (analysis.cpp:111-119) and uses_uv (analysis.cpp:148-154).
    const Graph& g = a.graph;
    const size_t n = g.nodes.size();
    a.dep.resize(n);
    a.uses_uv.resize(n);
    for (uint32_t id = 0; id < n; ++id) {
        uint8_t d = info(g.nodes[id].kind).dep;
        uint8_t uv = info(g.nodes[id].kind).dep == 1;
        for (uint32_t in : g.nodes[id].in) {
            d = std::max(d, a.dep[in]);
            uv = uv || a.uses_uv[in];
        }
        a.dep[id] = d;
        a.uses_uv[id] = uv;
    }

    // select_cache_points (analysis.cpp:121-139): a node is maximal when no
    // consumer chain reaches a cacheable node.
    std::vector<uint8_t> covered(n, 0);
    for (uint32_t id = static_cast<uint32_t>(n); id-- > 0;) {
        if (!covered[id] && a.dep[id] == 2) continue;
        for (uint32_t in : g.nodes[id].in) covered[in] = 1;
    }
    for (uint32_t id = 0; id < n; ++id) {
        if (a.dep[id] == 2 || covered[id]) continue;
        if (closure_size(g, id) < static_cast<size_t>(min_subtree_size)) continue;
        a.points.push_back(id);
    }
    return a;
}

std::string analysis_json(const Analysis& a) {
    static const char* kDep[] = {"const", "uv", "other"};
    json doc;
    doc["material_id"] = a.graph.material_id;
    doc["node_count"] = a.graph.nodes.size();
    json dep = json::array();
    for (uint32_t id = 0; id < a.graph.nodes.size(); ++id) {
        dep.push_back({{"id", id},
                       {"kind", std::string(kind_label(a.graph.nodes[id].kind))},
                       {"dep", kDep[a.dep[id]]}});
    }
    doc["dep"] = std::move(dep);
    json pts = json::array();
    for (uint32_t p : a.points) {
        pts.push_back({{"node", p},
                       {"uses_uv", static_cast<bool>(a.uses_uv[p])},
                       {"subtree_size", closure_size(a.graph, p)}});
    }
    doc["cache_points"] = std::move(pts);
    return doc.dump(2);
}

// ---------------------------------------------------------------------------
// Compiler: post-order emission with [CacheLookup ... CacheStore] brackets.
// ---------------------------------------------------------------------------
namespace {

class Compiler {
public:
    Compiler(const Analysis& a, const std::vector<std::string>& refs, Program& out)
        : a_(a), refs_(refs), out_(out), bracket_(a.graph.nodes.size(), -1),
          scalar_(a.graph.nodes.size(), -1) {
        for (size_t i = 0; i < a.points.size(); ++i) bracket_[a.points[i]] = static_cast<int>(i);
    }

    void run() { visit(a_.graph.output, false); }

private:
    const Analysis& a_;
    const std::vector<std::string>& refs_;
    Program& out_;
    std::vector<int> bracket_;
    std::vector<int8_t> scalar_;

    // Static value tag of a node's result (stackvm.cpp:36-75).
    bool scalar_of(uint32_t id) {
        if (scalar_[id] >= 0) return scalar_[id] != 0;
        const GNode& n = a_.graph.nodes[id];
        bool s = false;
        switch (n.kind) {
            case Kind::ConstFloat: case Kind::Checker: case Kind::NoiseFbm: case Kind::Dot:
                s = true;
                break;
            case Kind::Uv: s = n.uv_channel != 0; break;
            case Kind::Add: case Kind::Sub: case Kind::Mul: case Kind::Div: case Kind::Mix:
            case Kind::Power:
                s = scalar_of(n.in[0]) && scalar_of(n.in[1]);
                break;
            case Kind::Clamp: case Kind::SinWave: case Kind::BsdfOutput:
                s = scalar_of(n.in[0]);
                break;
            default: s = false; break;
        }
        scalar_[id] = s ? 1 : 0;
        return s;
    }

    mcg_insn blank(uint8_t op) {
        mcg_insn ins{};
        ins.op = op;
        return ins;
    }

    void visit(uint32_t id, bool in_bracket) {
        if (bracket_[id] >= 0) {
            if (in_bracket) fail(MCG_ERR_COMPILE, "nested cache point at node " + std::to_string(id));
            const size_t at = out_.code.size();
            mcg_insn look = blank(MCG_OP_CACHE_LOOKUP);
            look.arg = id;
            look.bracket = static_cast<uint16_t>(bracket_[id]);
            look.flags = (a_.uses_uv[id] ? MCG_F_USES_UV : 0u) |
                         (scalar_of(id) ? MCG_F_SCALAR_RESULT : 0u);
            out_.code.push_back(look);
            emit(id, true);
            mcg_insn store = blank(MCG_OP_CACHE_STORE);
            store.arg = id;
            store.bracket = static_cast<uint16_t>(bracket_[id]);
            store.flags = a_.uses_uv[id] ? MCG_F_USES_UV : 0u;
            out_.code.push_back(store);
            out_.code[at].imm.i = static_cast<int32_t>(out_.code.size() - (at + 1));
            return;
        }
        emit(id, in_bracket);
    }

    void emit(uint32_t id, bool in_bracket) {
        const GNode& n = a_.graph.nodes[id];
        for (uint32_t in : n.in) visit(in, in_bracket);
        mcg_insn ins{};
        switch (n.kind) {
            case Kind::ConstFloat:
            case Kind::ConstColor: {
                ins.op = MCG_OP_PUSH_CONST;
                ins.arg = static_cast<uint32_t>(out_.consts.size());
                mcg_const c{{n.value.x, n.value.y, n.value.z}, n.value.scalar ? 1u : 0u};
                out_.consts.push_back(c);
                break;
            }
            case Kind::Uv:
                ins.op = MCG_OP_LOAD_UV;
                ins.flags = static_cast<uint8_t>(n.uv_channel << MCG_F_UV_SHIFT);
                break;
            case Kind::Position: ins.op = MCG_OP_LOAD_POSITION; break;
            case Kind::Normal: ins.op = MCG_OP_LOAD_NORMAL; break;
            case Kind::Incoming: ins.op = MCG_OP_LOAD_INCOMING; break;
            case Kind::TexImage: {
                ins.op = MCG_OP_TEX_SAMPLE;
                const auto it = std::find(refs_.begin(), refs_.end(), n.image);
                if (it == refs_.end()) fail(MCG_ERR_COMPILE, "texture not loaded: " + n.image);
                ins.arg = static_cast<uint32_t>(it - refs_.begin());
                ins.flags = n.wrap_clamp ? MCG_F_WRAP_CLAMP : 0u;
                break;
            }
            case Kind::Checker:
                ins.op = MCG_OP_CHECKER;
                ins.imm.f = n.checker_scale;
                break;
            case Kind::NoiseFbm:
                ins.op = MCG_OP_NOISE;
                ins.arg = static_cast<uint32_t>(out_.noise.size());
                out_.noise.push_back(n.noise);
                break;
            case Kind::Add: ins.op = MCG_OP_ADD; break;
            case Kind::Sub: ins.op = MCG_OP_SUB; break;
            case Kind::Mul: ins.op = MCG_OP_MUL; break;
            case Kind::Div: ins.op = MCG_OP_DIV; break;
            case Kind::Mix: ins.op = MCG_OP_MIX; break;
            case Kind::Clamp: ins.op = MCG_OP_CLAMP; break;
            case Kind::Dot: ins.op = MCG_OP_DOT; break;
            case Kind::SinWave: ins.op = MCG_OP_SIN_WAVE; break;
            case Kind::ColorRamp:
                ins.op = MCG_OP_RAMP;
                ins.arg = static_cast<uint32_t>(out_.ramps.size());
                out_.ramps.push_back(n.stops);
                break;
            case Kind::Power: ins.op = MCG_OP_POWER; break;
            case Kind::BsdfDiffuse: ins.op = MCG_OP_BSDF_DIFFUSE; break;
            case Kind::BsdfOutput: return;  // transparent
        }
        out_.code.push_back(ins);
    }
};

int depth_change(uint8_t op) {
    switch (op) {
        case MCG_OP_PUSH_CONST: case MCG_OP_LOAD_UV: case MCG_OP_LOAD_POSITION:
        case MCG_OP_LOAD_NORMAL: case MCG_OP_LOAD_INCOMING: case MCG_OP_TEX_SAMPLE:
        case MCG_OP_CHECKER: case MCG_OP_NOISE:
            return 1;
        case MCG_OP_ADD: case MCG_OP_SUB: case MCG_OP_MUL: case MCG_OP_DIV: case MCG_OP_DOT:
        case MCG_OP_POWER:
            return -1;
        case MCG_OP_MIX:
            return -2;
        default:
            return 0;
    }
}

}  // namespace

Program compile_analysis(const Analysis& a, const std::vector<std::string>& refs,
                         int stack_limit) {
    if (a.points.size() > 64) {
        fail(MCG_ERR_COMPILE, "material has " + std::to_string(a.points.size()) +
                                  " cache points; limit is 64");
    }
    Program p;
    p.material_id = a.graph.material_id;
    p.cache_point_count = static_cast<uint32_t>(a.points.size());
    p.tex_refs = refs;
    Compiler(a, refs, p).run();
    mcg_insn end{};
    end.op = MCG_OP_END;
    p.code.push_back(end);

    // Balance check over the miss path, including the reference's
    // "depth <= 0" test after zero-effect ops (stackvm.cpp:232-236), which
    // rejects programs that open with a CacheLookup.
    int depth = 0, peak = 0;
    for (const mcg_insn& ins : p.code) {
        if (ins.op == MCG_OP_END) break;
        depth += depth_change(ins.op);
        if (depth <= 0) fail(MCG_ERR_COMPILE, "stack underflow during compilation");
        peak = std::max(peak, depth);
    }
    if (depth != 1) {
        fail(MCG_ERR_COMPILE, "unbalanced stack effect: final depth " + std::to_string(depth));
    }
    if (peak > stack_limit) {
        fail(MCG_ERR_COMPILE, "stack depth " + std::to_string(peak) + " exceeds limit " +
                                  std::to_string(stack_limit));
    }
    p.max_stack = peak;
    schedule_program(p);
    return p;
}

void schedule_program(Program& p) {
    // On the miss path the operand-stack depth before every instruction is a
    // compile-time constant, and so is every slot's scalar/rgb tag; a hit
    // pushes exactly one value of the bracket's static tag where the subtree
    // would have left one. The device VM therefore addresses its stack with
    // uniform slot numbers and never carries tags at run time.
    std::vector<uint8_t> tag;  // per live slot: 1 = scalar
    uint8_t stores = 0;
    for (mcg_insn& ins : p.code) {
        const int d = static_cast<int>(tag.size());
        ins.sp = static_cast<uint8_t>(d);
        uint8_t t = 0;
        auto top = [&](int k) { return tag[d - k]; };  // k = 1 is the top
        switch (ins.op) {
            case MCG_OP_PUSH_CONST:
                tag.push_back(p.consts[ins.arg].scalar ? 1 : 0);
                t = tag.back() ? MCG_T_R : 0;
                break;
            case MCG_OP_LOAD_UV:
                tag.push_back(((ins.flags >> MCG_F_UV_SHIFT) & 3u) != 0);
                t = tag.back() ? MCG_T_R : 0;
                break;
            case MCG_OP_LOAD_POSITION: case MCG_OP_LOAD_NORMAL: case MCG_OP_LOAD_INCOMING:
            case MCG_OP_TEX_SAMPLE:
                tag.push_back(0);
                break;
            case MCG_OP_CHECKER: case MCG_OP_NOISE:
                tag.push_back(1);
                t = MCG_T_R;
                break;
            case MCG_OP_ADD: case MCG_OP_SUB: case MCG_OP_MUL: case MCG_OP_DIV:
            case MCG_OP_POWER: case MCG_OP_DOT: {
                const uint8_t ta = top(2), tb = top(1);
                const uint8_t r = ins.op == MCG_OP_DOT ? 1 : (ta && tb);
                tag.pop_back();
                tag.back() = r;
                t = (ta ? MCG_T_A : 0) | (tb ? MCG_T_B : 0) | (r ? MCG_T_R : 0);
                break;
            }
            case MCG_OP_MIX: {
                const uint8_t ta = top(3), tb = top(2), tc = top(1);
                const uint8_t r = ta && tb;
                tag.pop_back();
                tag.pop_back();
                tag.back() = r;
                t = (ta ? MCG_T_A : 0) | (tb ? MCG_T_B : 0) | (tc ? MCG_T_C : 0) |
                    (r ? MCG_T_R : 0);
                break;
            }
            case MCG_OP_CLAMP: case MCG_OP_SIN_WAVE: {
                const uint8_t ta = top(1);
                t = ta ? (MCG_T_A | MCG_T_R) : 0;
                break;
            }
            case MCG_OP_RAMP: {
                const uint8_t ta = top(1);
                tag.back() = 0;
                t = ta ? MCG_T_A : 0;
                break;
            }
            case MCG_OP_BSDF_DIFFUSE: {
                const uint8_t ta = top(1);
                tag.back() = 0;
                t = ta ? MCG_T_A : 0;
                break;
            }
            case MCG_OP_CACHE_LOOKUP:
                t = (ins.flags & MCG_F_SCALAR_RESULT) ? MCG_T_R : 0;
                break;
            case MCG_OP_CACHE_STORE:
                ins.store_ord = stores++;
                t = top(1) ? (MCG_T_A | MCG_T_R) : 0;
                break;
            case MCG_OP_END:
                t = top(1) ? (MCG_T_A | MCG_T_R) : 0;
                break;
        }
        ins.tags = t;
    }
}

std::string disassemble_program(const Program& p) {
    const size_t n = p.code.size();
    std::vector<int> label(n + 1, -1);
    int next = 0;
    for (size_t i = 0; i < n; ++i) {
        if (p.code[i].op != MCG_OP_CACHE_LOOKUP) continue;
        const size_t target = i + 1 + static_cast<size_t>(p.code[i].imm.i);
        if (label[target] < 0) label[target] = next++;
    }
    std::ostringstream os;
    os << "material " << p.material_id << ", " << n << " instructions, max_stack " << p.max_stack
       << "\n";
    static const char* kPlain[] = {nullptr, nullptr, "load_position", "load_normal",
                                   "load_incoming", nullptr, nullptr, nullptr, "add", "sub",
                                   "mul", "div", "mix", "clamp", "dot", "sin_wave", nullptr,
                                   "power", "bsdf_diffuse", nullptr, nullptr, "end"};
    for (size_t i = 0; i < n; ++i) {
        if (label[i] >= 0) os << "L" << label[i] << ":\n";
        const mcg_insn& ins = p.code[i];
        os << "  " << i << ": ";
        switch (ins.op) {
            case MCG_OP_PUSH_CONST: {
                const mcg_const& c = p.consts[ins.arg];
                if (c.scalar) os << "push_const " << c.v[0];
                else os << "push_const (" << c.v[0] << ", " << c.v[1] << ", " << c.v[2] << ")";
                break;
            }
            case MCG_OP_LOAD_UV: {
                const unsigned ch = (ins.flags >> MCG_F_UV_SHIFT) & 3u;
                os << "load_uv" << (ch == 1 ? ".u" : ch == 2 ? ".v" : "");
                break;
            }
            case MCG_OP_TEX_SAMPLE:
                os << "tex_sample \"" << p.tex_refs[ins.arg] << "\" "
                   << ((ins.flags & MCG_F_WRAP_CLAMP) ? "clamp" : "repeat");
                break;
            case MCG_OP_CHECKER: os << "checker scale=" << ins.imm.f; break;
            case MCG_OP_NOISE: {
                const mcg_noise& z = p.noise[ins.arg];
                os << "noise octaves=" << z.octaves << " freq=" << z.frequency
                   << " lac=" << z.lacunarity << " gain=" << z.gain;
                break;
            }
            case MCG_OP_RAMP:
                os << "ramp #" << ins.arg << " (" << p.ramps[ins.arg].size() << " stops)";
                break;
            case MCG_OP_CACHE_LOOKUP:
                os << "cache_lookup node=" << ins.arg << " bracket=" << ins.bracket
                   << ((ins.flags & MCG_F_USES_UV) ? " uv" : " const") << " -> L"
                   << label[i + 1 + static_cast<size_t>(ins.imm.i)];
                break;
            case MCG_OP_CACHE_STORE:
                os << "cache_store node=" << ins.arg << " bracket=" << ins.bracket;
                break;
            default:
                os << kPlain[ins.op];
                break;
        }
        os << "\n";
    }
    return os.str();
}

}  // namespace mcg

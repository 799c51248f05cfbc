// Host-side runtime of libmcg: material graphs, analysis, compiler, scene
// preparation. Everything here runs once per scene on the CPU and produces the
// device layout declared in include/mcg.h. Reference behaviour is cited per
// function (paths relative to /root/reference/proj/core).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/mcg.h"

namespace mcg {

// An error that crosses the C ABI as a status code + message.
struct Failure : std::runtime_error {
    mcg_status code;
    Failure(mcg_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(mcg_status code, const std::string& msg) { throw Failure(code, msg); }

// Records the message for mcg_last_error() on this thread.
void set_last_error(const std::string& msg);
void clear_last_error();

// Runs `body`, converting exceptions to a status (the C ABI never throws).
template <typename F>
mcg_status guarded(F&& body) {
    try {
        clear_last_error();
        body();
        return MCG_OK;
    } catch (const Failure& f) {
        set_last_error(f.what());
        return f.code;
    } catch (const std::bad_alloc&) {
        set_last_error("out of host memory");
        return MCG_ERR_INVALID_ARGUMENT;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return MCG_ERR_INVALID_ARGUMENT;
    }
}

// ---------------------------------------------------------------------------
// Material graph (graph.hpp:20-86), node kinds in reference order.
// ---------------------------------------------------------------------------
enum class Kind : uint8_t {
    ConstFloat, ConstColor, Uv, Position, Normal, Incoming, TexImage, Checker, NoiseFbm,
    Add, Sub, Mul, Div, Mix, Clamp, Dot, SinWave, ColorRamp, Power, BsdfDiffuse, BsdfOutput,
};

// Host Value (value.hpp:25-63): scalars are stored replicated.
struct HVal {
    float x = 0, y = 0, z = 0;
    bool scalar = true;
    static HVal s(float v) { return {v, v, v, true}; }
    static HVal c(float r, float g, float b) { return {r, g, b, false}; }
    float lum() const { return scalar ? x : 0.2126f * x + 0.7152f * y + 0.0722f * z; }
};

struct GNode {
    Kind kind = Kind::ConstFloat;
    std::vector<uint32_t> in;
    HVal value;                 // ConstFloat / ConstColor
    int uv_channel = 0;         // 0 uv, 1 u, 2 v
    std::string image;          // TexImage
    bool wrap_clamp = false;    // TexImage
    float checker_scale = 1.0f; // Checker
    mcg_noise noise{4, 1.0f, 2.0f, 0.5f};
    std::vector<mcg_ramp_stop> stops;  // ColorRamp
};

struct Graph {
    uint32_t material_id = 0;
    std::vector<GNode> nodes;
    uint32_t output = 0;
};

int arity(Kind k);
const char* kind_label(Kind k);

// load_graph (graph.cpp:242-287) + validate_graph (graph.cpp:297-333).
Graph parse_graph(const std::string& json_text);
void check_graph(const Graph& g);

// analyze (analysis.cpp:141-156): folded graph, dependence classes,
// maximal cache points, uses_uv.
struct Analysis {
    Graph graph;
    std::vector<uint8_t> dep;          // 0 Const, 1 Uv, 2 Other
    std::vector<uint32_t> points;      // ascending
    std::vector<uint8_t> uses_uv;
    std::vector<uint32_t> remap;
};
Analysis analyze_graph(const Graph& g, int min_subtree_size);
std::string analysis_json(const Analysis& a);

// A compiled material in device layout: its instruction words and pools
// (the pools are per program here; flatten() concatenates them).
struct HostTexture {
    std::string ref;
    int width = 0, height = 0;
    std::vector<float> rgba;  // 4 floats per texel
};

struct Program {
    uint32_t material_id = 0;
    std::vector<mcg_insn> code;
    std::vector<mcg_const> consts;
    std::vector<mcg_noise> noise;
    std::vector<std::vector<mcg_ramp_stop>> ramps;
    std::vector<std::string> tex_refs;   // per TexSample arg (texture id -> ref)
    int max_stack = 0;
    uint32_t cache_point_count = 0;
};

// compile (stackvm.cpp:210-246) with the emitter (stackvm.cpp:15-174); a
// TexSample's texture id is its index in `loaded_refs` (the scene's pool).
Program compile_analysis(const Analysis& a, const std::vector<std::string>& loaded_refs,
                         int stack_limit = 256);
// Same listing as disassemble() (stackvm.cpp:370-443).
std::string disassemble_program(const Program& p);
// Annotates sp / tags / store_ord (the static stack schedule).
void schedule_program(Program& p);

// PPM reader (image.cpp:102-126) into RGBA floats.
HostTexture read_ppm_texture(const std::string& path, const std::string& ref);

}  // namespace mcg

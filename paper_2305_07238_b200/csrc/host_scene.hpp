// Prepared-scene container shared by the host loader and the device upload.
#pragma once

#include <string>
#include <vector>

#include "host_internal.hpp"

namespace mcg {

struct MeshData {
    std::vector<float> positions;  // 3 per vertex
    std::vector<float> uvs;        // 2 per vertex
    std::vector<uint32_t> indices;
    uint32_t material_id = 0;
};

struct SceneData {
    float cam_position[3] = {0, 0, 0};
    float cam_look_at[3] = {0, 0, -1};
    float cam_up[3] = {0, 1, 0};
    float cam_vfov_deg = 45.0f;
    int32_t cam_width = 256, cam_height = 256;
    float env[3] = {0, 0, 0};

    std::vector<MeshData> meshes;
    std::vector<mcg_sphere_in> spheres;
    std::vector<mcg_point_light> point_lights;
    std::vector<mcg_rect_light> rect_lights;

    std::vector<Analysis> analyses;   // empty when built from flat programs
    std::vector<Program> programs;    // per material slot
    std::vector<HostTexture> textures;

    // Flat device layout (include/mcg.h, mcg_flat_scene).
    std::vector<mcg_program> flat_programs;
    std::vector<mcg_insn> code;
    std::vector<mcg_const> consts;
    std::vector<mcg_noise> noise;
    std::vector<mcg_ramp> ramps;
    std::vector<mcg_ramp_stop> ramp_stops;
    std::vector<mcg_texture> tex_table;
    std::vector<float> texels;

    std::vector<mcg_bvh_node> nodes;
    std::vector<float> prim_geom;      // 12 per prim, leaf order
    std::vector<float> prim_uv;        // 6 per prim
    std::vector<uint32_t> prim_info;   // material slot | sphere flag
    std::vector<uint32_t> prim_source; // leaf position -> original primitive index
};

SceneData load_scene_file(const std::string& path, int min_subtree_size);
void prepare_scene(SceneData& s);
void flatten_programs(SceneData& s);
void fill_flat(const SceneData& s, mcg_flat_scene* f);
void camera_setup(const mcg_flat_scene& f, int32_t w, int32_t h, float out[12]);

}  // namespace mcg

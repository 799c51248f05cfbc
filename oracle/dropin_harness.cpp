// dropin_harness.cpp — TEST INFRASTRUCTURE. Drives the C++ drop-in
// (paper_2305_07238_b200/integration/matcache_render_b200.cpp) exactly as a
// reference caller would: matcache::load_scene (the reference's own loader,
// compiled in place) then matcache::render (now defined by the drop-in over
// libmcg). Built by `make -C oracle dropin` into oracle/_ref/libmcdropin.so.
#include <cstring>
#include <string>

#include "matcache/tracer.hpp"

extern "C" int dropin_render(const char* scene_path, int w, int h, int spp, int cache_on,
                             uint64_t n_cells, uint32_t n_entries, double* rad, double* nodes,
                             uint32_t* samples, uint64_t* stats_out, char* err, size_t cap) {
    try {
        const matcache::Scene scene = matcache::load_scene(scene_path);
        matcache::RenderConfig cfg;
        cfg.width = w;
        cfg.height = h;
        cfg.spp = spp;
        cfg.cache_enabled = cache_on != 0;
        cfg.n_cells = n_cells;
        cfg.n_entries = n_entries;
        const matcache::RenderResult r = matcache::render(scene, cfg);
        std::memcpy(rad, r.frame.radiance.data(), r.frame.radiance.size() * sizeof(double));
        std::memcpy(nodes, r.frame.nodes_found.data(), r.frame.nodes_found.size() * sizeof(double));
        std::memcpy(samples, r.frame.samples.data(), r.frame.samples.size() * sizeof(uint32_t));
        stats_out[0] = r.stats.lookups;
        stats_out[1] = r.stats.hits;
        stats_out[2] = r.stats.inserts_won;
        stats_out[3] = r.stats.inserts_lost_full;
        stats_out[4] = r.stats.instructions_executed;
        // exercise the experiment outputs too
        const matcache::DiffStats d = matcache::image_error(r.frame.radiance_image(),
                                                            r.frame.radiance_image());
        stats_out[5] = d.mean_abs == 0.0 ? 1 : 0;
        const matcache::StatsFile sf =
            matcache::parse_stats_json(matcache::stats_to_json(r.stats, r.frame));
        stats_out[6] = sf.per_pixel_nodes_found.size();
        return 0;
    } catch (const std::exception& e) {
        std::snprintf(err, cap, "%s", e.what());
        return 1;
    }
}

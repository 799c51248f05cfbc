// dropin_harness.cpp — TEST INFRASTRUCTURE. Drives the C++ drop-in
// (paper_2305_07238_b200/integration/matcache_render_b200.cpp) exactly as a
// reference caller would: matcache::load_scene (the reference's own loader,
// compiled in place) then matcache::render (now defined by the drop-in over
// libmcg). Built by `make -C oracle dropin` into oracle/_ref/libmcdropin.so.
#include <cstring>
#include <string>

#include "matcache/tracer.hpp"
#include "matcache_render_b200.hpp"

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

// Several scenes rendered one after the other, each loaded into a Scene that
// lives in the same stack slot (the pattern that defeats an address-keyed
// upload cache): radiance of render i at rad + i * w * h * 3. Cache off.
extern "C" int dropin_render_scenes(const char* const* paths, int n, int w, int h, int spp, double* rad,
                                    char* err, size_t cap) {
    try {
        for (int i = 0; i < n; ++i) {
            const matcache::Scene scene = matcache::load_scene(paths[i]);
            matcache::RenderConfig cfg;
            cfg.width = w;
            cfg.height = h;
            cfg.spp = spp;
            const matcache::RenderResult r = matcache::render(scene, cfg);
            std::memcpy(rad + static_cast<size_t>(i) * w * h * 3, r.frame.radiance.data(),
                        r.frame.radiance.size() * sizeof(double));
        }
        return 0;
    } catch (const std::exception& e) {
        std::snprintf(err, cap, "%s", e.what());
        return 1;
    }
}

// External caches through the drop-in: `renders` progressive renders into
// one heap MaterialCache, then the cache is deleted and a fresh one of the
// same shape (typically at the same address) rendered into once, then one
// of another shape. Per render, 6 numbers: stats lookups, hits, inserts_won,
// then the host table's occupied_slots(), counters().inserts_won, and
// whether its dump passes audit_dump (1/0). out[6 * (renders + 2)] and the
// next word: the first two caches' addresses.
extern "C" int dropin_render_external(const char* scene_path, int w, int h, int spp, uint64_t n_cells,
                                      uint32_t n_entries, int renders, const char* dump_path, uint64_t* out,
                                      char* err, size_t cap) {
    try {
        const matcache::Scene scene = matcache::load_scene(scene_path);
        matcache::RenderConfig cfg;
        cfg.width = w;
        cfg.height = h;
        cfg.spp = spp;
        cfg.cache_enabled = true;
        auto one = [&](matcache::MaterialCache* c, uint64_t* o) {
            cfg.n_cells = c->n_cells();
            cfg.n_entries = c->n_entries();
            const matcache::RenderResult r = matcache::render(scene, cfg, c);
            o[0] = r.stats.lookups;
            o[1] = r.stats.hits;
            o[2] = r.stats.inserts_won;
            o[3] = c->occupied_slots();
            o[4] = c->counters().inserts_won;
            c->dump(dump_path);
            o[5] = matcache::audit_dump(dump_path).clean ? 1 : 0;
        };
        auto* c = new matcache::MaterialCache(n_cells, n_entries);
        for (int i = 0; i < renders; ++i) one(c, out + 6 * i);
        out[6 * (renders + 2)] = reinterpret_cast<uintptr_t>(c);
        delete c;
        c = new matcache::MaterialCache(n_cells, n_entries);
        out[6 * (renders + 2) + 1] = reinterpret_cast<uintptr_t>(c);
        one(c, out + 6 * renders);
        delete c;
        c = new matcache::MaterialCache(n_cells / 2 + 1, n_entries > 1 ? n_entries - 1 : 1);
        one(c, out + 6 * (renders + 1));
        matcache::b200_release_cache(c);
        delete c;
        return 0;
    } catch (const std::exception& e) {
        std::snprintf(err, cap, "%s", e.what());
        return 1;
    }
}

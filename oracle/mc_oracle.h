/*
 * mc_oracle.h — TEST INFRASTRUCTURE ONLY. CPU restatement (plain C11) of the
 * reference's hot path: descriptor hashing, RGBE codec, Eq. 1 mip level,
 * texel indices, ray-cone footprint, counter RNG, node kernels, the stack-VM
 * interpreter over the flattened bytecode, the Nc x Ne first-insert-wins
 * table, BVH queries and the restated render().
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library, and only as the checker. The product path
 * (paper_2305_07238_b200/) never links or calls it.
 *
 * Pinning: each function is checked against the reference's own code,
 * compiled in place into oracle/_ref/libmcref.so (tests/test_oracle_vs_ref.py),
 * and against the committed fixtures in tests/golden/ generated from it
 * (tests/golden/make_golden.py).
 */
#ifndef MC_ORACLE_H_
#define MC_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#include "../include/mcg.h"

#ifdef __cplusplus
extern "C" {
#endif

uint64_t mco_hash_cell(const mcg_descriptor* d);
uint32_t mco_hash_check(const mcg_descriptor* d);
uint32_t mco_encode(const float rgb[3]);
void mco_decode(uint32_t packed, float rgb[3]);
uint8_t mco_mip_level(const float g1[2], const float g2[2], int mip_offset);
void mco_texel(const float uv[2], uint8_t level, uint32_t out[2]);
/* in: width, incoming[3], normal[3], e1[3], e2[3], duv1[2], duv2[2]; out g1, g2 */
void mco_footprint(const float in[17], float out[4]);
float mco_rng(uint64_t seed, uint64_t pixel, uint64_t sample, uint32_t dim);
float mco_perlin(float x, float y);
float mco_fbm(const mcg_noise* p, float u, float v);
float mco_sin_wave(float x);
float mco_power(float x, float y);

/* Batch wrappers for ctypes. */
void mco_hash_batch(const mcg_descriptor* d, size_t n, uint64_t* cell, uint32_t* check);
void mco_encode_batch(const float* rgb, size_t n, uint32_t* out);
void mco_decode_batch(const uint32_t* in, size_t n, float* rgb);
void mco_mip_texel_batch(const float* uv, const float* g1, const float* g2, size_t n, int off,
                         uint8_t* mip, uint32_t* txy);
void mco_footprint_batch(const float* in, size_t n, float* out);
void mco_fbm_batch(const int32_t* octaves, const float* fp, const float* uv, size_t n, float* out);
void mco_sin_wave_batch(const float* x, size_t n, float* out);
void mco_power_batch(const float* x, const float* y, size_t n, float* out);
void mco_atan2f_batch(const float* y, const float* x, size_t n, float* out);
void mco_acosf_batch(const float* x, size_t n, float* out);

/* The table (cache.cpp semantics; single-threaded). */
typedef struct mco_cache mco_cache;
mco_cache* mco_cache_new(uint64_t n_cells, uint32_t n_entries);
void mco_cache_free(mco_cache* c);
/* returns outcome (MCG_INSERT_*) */
int mco_cache_update(mco_cache* c, const mcg_descriptor* d, const float rgb[3], uint64_t* slot,
                     uint64_t* packed);
int mco_cache_lookup(mco_cache* c, const mcg_descriptor* d, float rgb[3]);
void mco_cache_update_batch(mco_cache* c, const mcg_descriptor* d, const float* rgb, size_t n,
                            uint8_t* outcome, uint64_t* slot, uint64_t* packed);
void mco_cache_lookup_batch(mco_cache* c, const mcg_descriptor* d, size_t n, uint8_t* hit,
                            float* rgb);
const uint64_t* mco_cache_slots(const mco_cache* c);
void mco_cache_counters(const mco_cache* c, uint64_t out[5]);

/* execute (stackvm.cpp:248-368) over the flattened program of `slot`.
 * sp: position, normal, incoming, uv, g1, g2 (15 floats). value_out: rgb +
 * tag word. cache may be NULL (binding disabled). */
void mco_execute_batch(const mcg_flat_scene* s, uint32_t slot, const float* sp, size_t n,
                       mco_cache* cache, int mip_offset, float* values, uint32_t* nodes,
                       uint32_t* instrs);

/* Deterministic-mode batch: lookups see the table as it was at the call;
 * the stores are applied afterwards in (point index, store ordinal) order
 * (mcg_execute_batch with MCG_CACHE_DETERMINISTIC). */
void mco_execute_batch_deferred(const mcg_flat_scene* s, uint32_t slot, const float* sp, size_t n,
                                mco_cache* cache, int mip_offset, float* values, uint32_t* nodes,
                                uint32_t* instrs);

/* Scene::intersect (scene.cpp:252-278) on the flat BVH; out 24 floats per ray
 * in the harness layout (found, t, position, normal, uv, slot, e1, e2, duv1, duv2). */
void mco_intersect_batch(const mcg_flat_scene* s, const float* rays, size_t n, float t_min,
                         float t_max, float* out);
void mco_occluded_batch(const mcg_flat_scene* s, const float* rays, size_t n, float t_min,
                        const float* t_max, uint8_t* out);

/* render() restated. mode: 0 cache off, 1 epoch-sequential (immediate
 * inserts: the reference update() in (sample, bounce, pixel) order),
 * 3 deterministic (epoch-deferred inserts applied in (pixel, store) order). */
typedef struct mco_render_params {
    int32_t width, height, spp, max_bounces;
    int32_t mode;
    int32_t mip_offset;
    uint64_t n_cells;
    uint32_t n_entries;
    uint32_t first_sample;
    uint64_t rng_seed;
    float diffuse_spread;
    int32_t tile_size;
    int32_t shard_rank, shard_count, shard_mode;
    int32_t threads;
    int32_t samples_per_pass;  /* samples per wavefront pass (0 -> 1); the epoch
                                  of deterministic mode is one (pass, bounce) */
} mco_render_params;

typedef struct mco_render_stats {
    double wall_time_s;
    uint64_t lookups, hits, inserts_won, inserts_lost_full;
    uint64_t stores_attempted, stores_won, instructions_executed;
    uint64_t paths, shading_points;
} mco_render_stats;

/* camera: the 12 floats of mcg_camera_setup, computed here independently. */
void mco_camera_setup(const mcg_flat_scene* s, int w, int h, float out[12]);
int mco_render(const mcg_flat_scene* s, const mco_render_params* p, mco_cache* external_cache,
               double* radiance, double* nodes_found, uint32_t* samples,
               uint64_t* hits_per_sample, mco_render_stats* stats);

#ifdef __cplusplus
}
#endif

#endif /* MC_ORACLE_H_ */

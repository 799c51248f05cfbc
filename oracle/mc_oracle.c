/*
 * mc_oracle.c — TEST INFRASTRUCTURE ONLY (see mc_oracle.h). A deliberately
 * plain, scalar C restatement of the reference algorithm, written for
 * readability against the cited reference lines (paths relative to
 * /root/reference/proj/core), not for speed.
 *
 * Compiled with -ffp-contract=off like the reference (proj/CMakeLists.txt:16).
 */
#define _GNU_SOURCE
#include "mc_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "mc_detmath.h"

/* ---------------------------------------------------------------- rng.hpp */

/* mix64: include/matcache/rng.hpp:8-13 */
static uint64_t mix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

/* PathRng: rng.hpp:18-31 */
typedef struct { uint64_t key; } Rng;
static Rng rng_make(uint64_t seed, uint64_t pixel, uint64_t sample) {
    Rng r;
    r.key = mix64(seed ^ mix64(pixel ^ mix64(sample)));
    return r;
}
static float rng_sample(Rng r, uint32_t dim) {
    const uint64_t h = mix64(r.key + 0x632be59bd9b4e019ull * (uint64_t)(dim + 1));
    return (float)(h >> 40) * 0x1.0p-24f;
}
float mco_rng(uint64_t seed, uint64_t pixel, uint64_t sample, uint32_t dim) {
    return rng_sample(rng_make(seed, pixel, sample), dim);
}

/* -------------------------------------------------------------- cache.cpp */

/* hash_descriptor: src/cache.cpp:21-30 */
static uint64_t hash_descriptor(const mcg_descriptor* d, uint64_t seed) {
    const uint64_t w0 = (uint64_t)d->mat_idx | ((uint64_t)d->node_idx << 32);
    const uint64_t w1 = (uint64_t)d->texel_x | ((uint64_t)d->texel_y << 32);
    const uint64_t w2 = d->mip_level;
    uint64_t h = seed;
    h = mix64(h ^ w0);
    h = mix64(h ^ w1);
    h = mix64(h ^ w2);
    return h;
}
/* hash_cell / hash_check: src/cache.cpp:34-39 */
uint64_t mco_hash_cell(const mcg_descriptor* d) { return hash_descriptor(d, 0x243f6a8885a308d3ull); }
uint32_t mco_hash_check(const mcg_descriptor* d) {
    const uint32_t h = (uint32_t)hash_descriptor(d, 0x13198a2e03707344ull);
    return h == 0 ? 1u : h;
}

/* encode_value: src/cache.cpp:41-61 */
uint32_t mco_encode(const float v[3]) {
    const double r = (isfinite(v[0]) && v[0] > 0.0f) ? v[0] : 0.0;
    const double g = (isfinite(v[1]) && v[1] > 0.0f) ? v[1] : 0.0;
    const double b = (isfinite(v[2]) && v[2] > 0.0f) ? v[2] : 0.0;
    const double d = fmax(r, fmax(g, b));
    if (d <= 0.0) return 0;
    int e = 0;
    (void)frexp(d, &e);
    if (e < -127) return 0;
    if (e > 127) e = 127;
    const double fac = ldexp(256.0, -e);
    uint32_t mr = (uint32_t)(r * fac), mg = (uint32_t)(g * fac), mb = (uint32_t)(b * fac);
    if (mr > 255) mr = 255;
    if (mg > 255) mg = 255;
    if (mb > 255) mb = 255;
    return ((uint32_t)(e + 128) << 24) | (mr << 16) | (mg << 8) | mb;
}

/* decode_value: src/cache.cpp:63-71 */
void mco_decode(uint32_t packed, float out[3]) {
    const uint32_t ex = packed >> 24;
    if (ex == 0) {
        out[0] = out[1] = out[2] = 0.0f;
        return;
    }
    const double scale = ldexp(1.0, (int)ex - 128 - 8);
    out[0] = (float)((((packed >> 16) & 255u) + 0.5) * scale);
    out[1] = (float)((((packed >> 8) & 255u) + 0.5) * scale);
    out[2] = (float)(((packed & 255u) + 0.5) * scale);
}

struct mco_cache {
    uint64_t n_cells;
    uint32_t n_entries;
    uint64_t* slots;
    uint64_t lookups, hits, won, lost_full;
};

mco_cache* mco_cache_new(uint64_t n_cells, uint32_t n_entries) {
    if (n_cells == 0 || n_entries == 0) return NULL;
    mco_cache* c = (mco_cache*)calloc(1, sizeof(mco_cache));
    c->n_cells = n_cells;
    c->n_entries = n_entries;
    c->slots = (uint64_t*)calloc(n_cells * n_entries, sizeof(uint64_t));
    return c;
}
void mco_cache_free(mco_cache* c) {
    if (!c) return;
    free(c->slots);
    free(c);
}
const uint64_t* mco_cache_slots(const mco_cache* c) { return c->slots; }
void mco_cache_counters(const mco_cache* c, uint64_t out[5]) {
    out[0] = c->lookups;
    out[1] = c->hits;
    out[2] = c->won;
    out[3] = c->lost_full;
    uint64_t occ = 0;
    for (uint64_t i = 0; i < c->n_cells * c->n_entries; ++i) occ += c->slots[i] != 0;
    out[4] = occ;
}

/* MaterialCache::update: src/cache.cpp:94-119 (single thread: the CAS from
 * zero always succeeds, so LostRace cannot occur here). */
static int cache_update_hashed(mco_cache* c, uint64_t cell_hash, uint32_t check, uint32_t payload,
                               uint64_t* slot_out, uint64_t* packed_out) {
    const uint64_t base = (cell_hash % c->n_cells) * c->n_entries;
    for (uint32_t i = 0; i < c->n_entries; ++i) {
        const uint64_t cur = c->slots[base + i];
        if ((uint32_t)(cur >> 32) == check) {
            if (slot_out) *slot_out = base + i;
            if (packed_out) *packed_out = cur;
            return MCG_INSERT_ALREADY_PRESENT;
        }
        if (cur == 0) {
            const uint64_t packed = ((uint64_t)check << 32) | payload;
            c->slots[base + i] = packed;
            c->won++;
            if (slot_out) *slot_out = base + i;
            if (packed_out) *packed_out = packed;
            return MCG_INSERT_WON;
        }
    }
    c->lost_full++;
    if (slot_out) *slot_out = ~(uint64_t)0;
    if (packed_out) *packed_out = 0;
    return MCG_INSERT_CELL_FULL;
}

int mco_cache_update(mco_cache* c, const mcg_descriptor* d, const float rgb[3], uint64_t* slot,
                     uint64_t* packed) {
    return cache_update_hashed(c, mco_hash_cell(d), mco_hash_check(d), mco_encode(rgb), slot, packed);
}

/* MaterialCache::lookup: src/cache.cpp:121-136 */
int mco_cache_lookup(mco_cache* c, const mcg_descriptor* d, float rgb[3]) {
    c->lookups++;
    const uint64_t base = (mco_hash_cell(d) % c->n_cells) * c->n_entries;
    const uint32_t check = mco_hash_check(d);
    for (uint32_t i = 0; i < c->n_entries; ++i) {
        const uint64_t cur = c->slots[base + i];
        if (cur == 0) return 0;
        if ((uint32_t)(cur >> 32) == check) {
            c->hits++;
            mco_decode((uint32_t)cur, rgb);
            return 1;
        }
    }
    return 0;
}

void mco_cache_update_batch(mco_cache* c, const mcg_descriptor* d, const float* rgb, size_t n,
                            uint8_t* outcome, uint64_t* slot, uint64_t* packed) {
    for (size_t i = 0; i < n; ++i) {
        uint64_t s, p;
        const int o = mco_cache_update(c, &d[i], rgb + 3 * i, &s, &p);
        if (outcome) outcome[i] = (uint8_t)o;
        if (slot) slot[i] = s;
        if (packed) packed[i] = p;
    }
}
void mco_cache_lookup_batch(mco_cache* c, const mcg_descriptor* d, size_t n, uint8_t* hit,
                            float* rgb) {
    for (size_t i = 0; i < n; ++i) {
        float v[3] = {0, 0, 0};
        hit[i] = (uint8_t)mco_cache_lookup(c, &d[i], v);
        memcpy(rgb + 3 * i, v, sizeof(v));
    }
}

/* ------------------------------------------------------------ raycone.cpp */

typedef struct { float x, y, z; } V3;
typedef struct { float x, y; } V2;

static V3 v3_add(V3 a, V3 b) { V3 r = {a.x + b.x, a.y + b.y, a.z + b.z}; return r; }
static V3 v3_sub(V3 a, V3 b) { V3 r = {a.x - b.x, a.y - b.y, a.z - b.z}; return r; }
static V3 v3_mul(V3 a, float s) { V3 r = {a.x * s, a.y * s, a.z * s}; return r; }
static V3 v3_hadamard(V3 a, V3 b) { V3 r = {a.x * b.x, a.y * b.y, a.z * b.z}; return r; }
static float v3_dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static V3 v3_cross(V3 a, V3 b) {
    V3 r = {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
    return r;
}
static float v3_len(V3 a) { return sqrtf(v3_dot(a, a)); }
/* normalize: include/matcache/geom.hpp:34-37 */
static V3 v3_norm(V3 a) {
    const float len = v3_len(a);
    if (len > 0.0f) return v3_mul(a, 1.0f / len);
    V3 z = {0, 0, 0};
    return z;
}
static V3 v3_load(const float* p) { V3 r = {p[0], p[1], p[2]}; return r; }
static float v2_len(V2 a) { return sqrtf(a.x * a.x + a.y * a.y); }

/* mip_level: src/raycone.cpp:67-73. floor(-log2(m)) is evaluated exactly
 * from the binary exponent: m = f 2^E, f in [0.5,1): -E+1 if f == 0.5 else -E
 * (bit-identical to floor(-std::log2((double)m))). */
uint8_t mco_mip_level(const float g1[2], const float g2[2], int off) {
    V2 a = {g1[0], g1[1]}, b = {g2[0], g2[1]};
    const float m = fminf(v2_len(a), v2_len(b));
    if (!(m > 0.0f)) return 24;
    int32_t lv;
    if (isinf(m)) {
        /* floor(-log2(inf)) = -inf converts to INT_MIN on x86-64 (cvttsd2si),
         * and the reference's `+ mip_offset` then wraps: mirror that. */
        lv = (int32_t)(0x80000000u + (uint32_t)off);
    } else {
        int e;
        const double f = frexp((double)m, &e);
        lv = (f == 0.5 ? 1 - e : -e) + off;
    }
    return (uint8_t)(lv < 0 ? 0 : (lv > 24 ? 24 : lv));
}

/* texel_indices: src/raycone.cpp:75-83 */
void mco_texel(const float uv[2], uint8_t level, uint32_t out[2]) {
    const uint32_t res = 1u << level;
    for (int k = 0; k < 2; ++k) {
        const float t = uv[k];
        const float w = t - floorf(t);
        const float s = w * (float)res;
        uint32_t i = (s != s) ? 0u : (uint32_t)s;
        out[k] = i >= res ? res - 1 : i;
    }
}

/* world_to_uv: src/raycone.cpp:35-46 */
static V2 world_to_uv(V3 a, V3 e1, V3 e2, V2 duv1, V2 duv2) {
    const float g11 = v3_dot(e1, e1), g12 = v3_dot(e1, e2), g22 = v3_dot(e2, e2);
    const float det = g11 * g22 - g12 * g12;
    V2 r = {0.0f, 0.0f};
    if (fabsf(det) < 1e-20f) return r;
    const float r1 = v3_dot(a, e1), r2 = v3_dot(a, e2);
    const float alpha = (r1 * g22 - r2 * g12) / det;
    const float beta = (r2 * g11 - r1 * g12) / det;
    r.x = duv1.x * alpha + duv2.x * beta;
    r.y = duv1.y * alpha + duv2.y * beta;
    return r;
}

/* footprint_gradients: src/raycone.cpp:50-65 (any_tangent :28-31) */
static void footprint(float width, V3 inc, V3 n, V3 e1, V3 e2, V2 duv1, V2 duv2, V2* g1, V2* g2) {
    const float cos_t = fmaxf(fabsf(v3_dot(inc, n)), 1e-4f);
    const V3 proj = v3_sub(inc, v3_mul(n, v3_dot(inc, n)));
    const float plen = v3_len(proj);
    V3 ax1;
    if (plen > 1e-6f) {
        ax1 = v3_mul(proj, 1.0f / plen);
    } else {
        V3 axis = {1, 0, 0};
        if (!(fabsf(n.x) < 0.9f)) { axis.x = 0; axis.y = 1; }
        ax1 = v3_norm(v3_cross(n, axis));
    }
    const V3 ax2 = v3_norm(v3_cross(n, ax1));
    const float half_major = width / (2.0f * cos_t);
    const float half_minor = width * 0.5f;
    *g1 = world_to_uv(v3_mul(ax1, half_major), e1, e2, duv1, duv2);
    *g2 = world_to_uv(v3_mul(ax2, half_minor), e1, e2, duv1, duv2);
}

void mco_footprint(const float in[17], float out[4]) {
    V2 g1, g2;
    V2 d1 = {in[13], in[14]}, d2 = {in[15], in[16]};
    footprint(in[0], v3_load(in + 1), v3_load(in + 4), v3_load(in + 7), v3_load(in + 10), d1, d2,
              &g1, &g2);
    out[0] = g1.x;
    out[1] = g1.y;
    out[2] = g2.x;
    out[3] = g2.y;
}

/* -------------------------------------------------------------- noise.cpp */

/* Ken Perlin's reference permutation (src/noise.cpp:12-29). */
static const uint8_t kPerm[256] = {
    151, 160, 137, 91, 90, 15, 131, 13, 201, 95, 96, 53, 194, 233, 7, 225, 140, 36, 103, 30,
    69, 142, 8, 99, 37, 240, 21, 10, 23, 190, 6, 148, 247, 120, 234, 75, 0, 26, 197, 62, 94,
    252, 219, 203, 117, 35, 11, 32, 57, 177, 33, 88, 237, 149, 56, 87, 174, 20, 125, 136, 171,
    168, 68, 175, 74, 165, 71, 134, 139, 48, 27, 166, 77, 146, 158, 231, 83, 111, 229, 122, 60,
    211, 133, 230, 220, 105, 92, 41, 55, 46, 245, 40, 244, 102, 143, 54, 65, 25, 63, 161, 1,
    216, 80, 73, 209, 76, 132, 187, 208, 89, 18, 169, 200, 196, 135, 130, 116, 188, 159, 86,
    164, 100, 109, 198, 173, 186, 3, 64, 52, 217, 226, 250, 124, 123, 5, 202, 38, 147, 118,
    126, 255, 82, 85, 212, 207, 206, 59, 227, 47, 16, 58, 17, 182, 189, 28, 42, 223, 183, 170,
    213, 119, 248, 152, 2, 44, 154, 163, 70, 221, 153, 101, 155, 167, 43, 172, 9, 129, 22, 39,
    253, 19, 98, 108, 110, 79, 113, 224, 232, 178, 185, 112, 104, 218, 246, 97, 228, 251, 34,
    242, 193, 238, 210, 144, 12, 191, 179, 162, 241, 81, 51, 145, 235, 249, 14, 239, 107, 49,
    192, 214, 31, 181, 199, 106, 157, 184, 84, 204, 176, 115, 121, 50, 45, 127, 4, 150, 254,
    138, 236, 205, 93, 222, 114, 67, 29, 24, 72, 243, 141, 128, 195, 78, 66, 215, 61, 156, 180,
};

static int perm(int i) { return kPerm[i & 255]; }
static float fade(float t) { return t * t * t * (t * (t * 6.0f - 15.0f) + 10.0f); }
static float lerpf_(float a, float b, float t) { return a + (b - a) * t; }
static float grad2(int h, float dx, float dy) {
    switch (h & 7) {
        case 0: return dx + dy;
        case 1: return -dx + dy;
        case 2: return dx - dy;
        case 3: return -dx - dy;
        case 4: return dx;
        case 5: return -dx;
        case 6: return dy;
        default: return -dy;
    }
}

/* perlin2: src/noise.cpp:53-75 */
float mco_perlin(float x, float y) {
    const float fx = floorf(x), fy = floorf(y);
    const int ix = (int)fx, iy = (int)fy;
    const float dx = x - fx, dy = y - fy;
    const float u = fade(dx), v = fade(dy);
    const int a = perm(ix) + iy;
    const int b = perm(ix + 1) + iy;
    const float n00 = grad2(perm(a), dx, dy);
    const float n10 = grad2(perm(b), dx - 1.0f, dy);
    const float n01 = grad2(perm(a + 1), dx, dy - 1.0f);
    const float n11 = grad2(perm(b + 1), dx - 1.0f, dy - 1.0f);
    const float n = lerpf_(lerpf_(n00, n10, u), lerpf_(n01, n11, u), v);
    return n * 1.41421356f;
}

/* fbm2: src/noise.cpp:77-91 */
float mco_fbm(const mcg_noise* p, float u, float v) {
    int oct = p->octaves < 1 ? 1 : (p->octaves > 10 ? 10 : p->octaves);
    float sum = 0.0f, amp = 1.0f, norm = 0.0f, freq = p->frequency;
    for (int o = 0; o < oct; ++o) {
        sum += amp * mco_perlin(u * freq, v * freq);
        norm += amp;
        amp *= p->gain;
        freq *= p->lacunarity;
    }
    const float n = norm > 0.0f ? sum / norm : 0.0f;
    return fminf(fmaxf(0.5f + 0.5f * n, 0.0f), 1.0f);
}

/* ------------------------------------------------------------ texture.cpp */

static float wrap_coord(float t, int clamp) {
    if (!clamp) return t - floorf(t);
    return fminf(fmaxf(t, 0.0f), 1.0f);
}
static int wrap_index(int i, int n, int clamp) {
    if (!clamp) {
        i %= n;
        return i < 0 ? i + n : i;
    }
    return i < 0 ? 0 : (i >= n ? n - 1 : i);
}

/* sample_bilinear: src/texture.cpp:24-48 over RGBA texels */
static void bilinear(const mcg_flat_scene* s, uint32_t tex, float uu, float vv, int clamp,
                     float out[3]) {
    const mcg_texture* t = &s->textures[tex];
    const float* px = s->texels + 4 * t->offset;
    const float u = wrap_coord(uu, clamp), v = wrap_coord(vv, clamp);
    const float x = u * (float)t->width - 0.5f;
    const float y = v * (float)t->height - 0.5f;
    const float fx = floorf(x), fy = floorf(y);
    const float tx = x - fx, ty = y - fy;
    const int x0 = wrap_index((int)fx, t->width, clamp);
    const int x1 = wrap_index((int)fx + 1, t->width, clamp);
    const int y0 = wrap_index((int)fy, t->height, clamp);
    const int y1 = wrap_index((int)fy + 1, t->height, clamp);
    const float* c00 = px + 4 * ((size_t)y0 * t->width + x0);
    const float* c10 = px + 4 * ((size_t)y0 * t->width + x1);
    const float* c01 = px + 4 * ((size_t)y1 * t->width + x0);
    const float* c11 = px + 4 * ((size_t)y1 * t->width + x1);
    const float wx = 1.0f - tx, wy = 1.0f - ty;
    for (int k = 0; k < 3; ++k) {
        const float top = c00[k] * wx + c10[k] * tx;
        const float bot = c01[k] * wx + c11[k] * tx;
        out[k] = top * wy + bot * ty;
    }
}

/* checker: src/texture.cpp:50-54 */
static float checker(float scale, float u, float v) {
    const int iu = (int)floorf(u * scale);
    const int iv = (int)floorf(v * scale);
    return ((iu + iv) & 1) == 0 ? 1.0f : 0.0f;
}

/* ----------------------------------------------------- value.hpp: Value ops */

typedef struct { float x, y, z; int scalar; } Val;

static Val val_s(float s) { Val v = {s, s, s, 1}; return v; }
static Val val_c(float r, float g, float b) { Val v = {r, g, b, 0}; return v; }
/* as_scalar: value.hpp:36-38 */
static float val_lum(Val v) { return v.scalar ? v.x : 0.2126f * v.x + 0.7152f * v.y + 0.0722f * v.z; }

/* componentwise2: value.hpp:74-81 */
static Val lane2(Val a, Val b, int op, float t) {
    float ra[3] = {a.x, a.y, a.z}, rb[3] = {b.x, b.y, b.z}, r[3];
    for (int k = 0; k < 3; ++k) {
        const float x = ra[k], y = rb[k];
        switch (op) {
            case MCG_OP_ADD: r[k] = x + y; break;
            case MCG_OP_SUB: r[k] = x - y; break;
            case MCG_OP_MUL: r[k] = x * y; break;
            case MCG_OP_DIV: r[k] = y == 0.0f ? 0.0f : x / y; break; /* :106-108 */
            case MCG_OP_MIX: r[k] = x * (1.0f - t) + y * t; break;     /* :110-113 */
            default: { /* MCG_OP_POWER, :132-137 */
                const float p = mc_powf_nonneg(fmaxf(x, 0.0f), y);
                r[k] = isfinite(p) ? p : 0.0f;
            }
        }
    }
    return (a.scalar && b.scalar) ? val_s(r[0]) : val_c(r[0], r[1], r[2]);
}

float mco_sin_wave(float x) { return 0.5f + 0.5f * mc_sinf(x * 6.28318530717958647692f); }
float mco_power(float x, float y) {
    const float p = mc_powf_nonneg(fmaxf(x, 0.0f), y);
    return isfinite(p) ? p : 0.0f;
}

/* componentwise1: value.hpp:83-88 (clamp01 :115-117, sin_wave :125-128) */
static Val lane1(Val a, int op) {
    float ra[3] = {a.x, a.y, a.z}, r[3];
    for (int k = 0; k < 3; ++k) {
        r[k] = op == MCG_OP_CLAMP ? fminf(fmaxf(ra[k], 0.0f), 1.0f) : mco_sin_wave(ra[k]);
    }
    return a.scalar ? val_s(r[0]) : val_c(r[0], r[1], r[2]);
}

/* ramp: value.hpp:141-156 */
static Val ramp(const mcg_flat_scene* s, uint32_t ri, Val fac) {
    const mcg_ramp* rp = &s->ramps[ri];
    const mcg_ramp_stop* st = s->ramp_stops + rp->first;
    const uint32_t n = rp->count;
    if (n == 0) return val_c(0, 0, 0);
    const float t = val_lum(fac);
    if (t <= st[0].t) return val_c(st[0].r, st[0].g, st[0].b);
    if (t >= st[n - 1].t) return val_c(st[n - 1].r, st[n - 1].g, st[n - 1].b);
    for (uint32_t i = 1; i < n; ++i) {
        if (t <= st[i].t) {
            const float span = st[i].t - st[i - 1].t;
            const float w = span > 0.0f ? (t - st[i - 1].t) / span : 0.0f;
            const float u = 1.0f - w;
            return val_c(st[i - 1].r * u + st[i].r * w, st[i - 1].g * u + st[i].g * w,
                         st[i - 1].b * u + st[i].b * w);
        }
    }
    return val_c(st[n - 1].r, st[n - 1].g, st[n - 1].b);
}

/* ---------------------------------------------------------- stackvm.cpp VM */

typedef struct {
    float pos[3], nrm[3], inc[3], uv[2], g1[2], g2[2];
} ShadePt;

typedef struct {
    uint64_t cell_hash;
    uint32_t check;
    uint32_t payload;
    uint32_t key;
} PendingStore;

typedef struct {
    mco_cache* cache;      /* NULL: binding disabled */
    int mip_offset;
    int deferred;          /* deterministic mode: stores go to the queue */
    PendingStore* queue;
    size_t queue_len, queue_cap;
    uint32_t key_base;     /* pixel << 6 */
    uint64_t stores_attempted, stores_won, instructions;
} Binding;

static void queue_push(Binding* b, PendingStore p) {
    if (b->queue_len == b->queue_cap) {
        b->queue_cap = b->queue_cap ? 2 * b->queue_cap : 1024;
        b->queue = (PendingStore*)realloc(b->queue, b->queue_cap * sizeof(PendingStore));
    }
    b->queue[b->queue_len++] = p;
}

/* execute: src/stackvm.cpp:248-368, over the flattened instruction words. */
static Val execute(const mcg_flat_scene* s, uint32_t slot, const ShadePt* sp, Binding* b,
                   uint32_t* nodes_found) {
    Val stack[256];
    mcg_descriptor pending[64];
    uint64_t pend_cell[64];
    uint32_t pend_check[64];
    int top = 0;
    const mcg_program* prog = &s->programs[slot];
    const mcg_insn* code = s->code + prog->code_offset;
    size_t pc = 0;
    for (;;) {
        const mcg_insn* ins = &code[pc++];
        b->instructions++;
        switch (ins->op) {
            case MCG_OP_PUSH_CONST: {
                const mcg_const* c = &s->consts[ins->arg];
                stack[top++] = c->scalar ? val_s(c->v[0]) : val_c(c->v[0], c->v[1], c->v[2]);
                break;
            }
            case MCG_OP_LOAD_UV: {
                const unsigned ch = (ins->flags >> MCG_F_UV_SHIFT) & 3u;
                stack[top++] = ch == 0 ? val_c(sp->uv[0], sp->uv[1], 0.0f)
                                       : val_s(ch == 1 ? sp->uv[0] : sp->uv[1]);
                break;
            }
            case MCG_OP_LOAD_POSITION: stack[top++] = val_c(sp->pos[0], sp->pos[1], sp->pos[2]); break;
            case MCG_OP_LOAD_NORMAL: stack[top++] = val_c(sp->nrm[0], sp->nrm[1], sp->nrm[2]); break;
            case MCG_OP_LOAD_INCOMING: stack[top++] = val_c(sp->inc[0], sp->inc[1], sp->inc[2]); break;
            case MCG_OP_TEX_SAMPLE: {
                float c[3];
                bilinear(s, ins->arg, sp->uv[0], sp->uv[1], (ins->flags & MCG_F_WRAP_CLAMP) != 0, c);
                stack[top++] = val_c(c[0], c[1], c[2]);
                break;
            }
            case MCG_OP_CHECKER: stack[top++] = val_s(checker(ins->imm.f, sp->uv[0], sp->uv[1])); break;
            case MCG_OP_NOISE: stack[top++] = val_s(mco_fbm(&s->noise[ins->arg], sp->uv[0], sp->uv[1])); break;
            case MCG_OP_ADD: case MCG_OP_SUB: case MCG_OP_MUL: case MCG_OP_DIV: case MCG_OP_POWER:
                stack[top - 2] = lane2(stack[top - 2], stack[top - 1], ins->op, 0.0f);
                --top;
                break;
            case MCG_OP_MIX:
                stack[top - 3] = lane2(stack[top - 3], stack[top - 2], MCG_OP_MIX, val_lum(stack[top - 1]));
                top -= 2;
                break;
            case MCG_OP_CLAMP: case MCG_OP_SIN_WAVE:
                stack[top - 1] = lane1(stack[top - 1], ins->op);
                break;
            case MCG_OP_DOT: { /* value.hpp:119-123 */
                const Val a = stack[top - 2], c = stack[top - 1];
                stack[top - 2] = val_s(a.x * c.x + a.y * c.y + a.z * c.z);
                --top;
                break;
            }
            case MCG_OP_RAMP: stack[top - 1] = ramp(s, ins->arg, stack[top - 1]); break;
            case MCG_OP_BSDF_DIFFUSE: {
                const Val a = stack[top - 1];
                stack[top - 1] = val_c(a.x, a.y, a.z);
                break;
            }
            case MCG_OP_CACHE_LOOKUP: { /* :328-349 */
                if (!b->cache) break;
                mcg_descriptor d;
                memset(&d, 0, sizeof(d));
                d.mat_idx = prog->material_id;
                d.node_idx = ins->arg;
                if (ins->flags & MCG_F_USES_UV) {
                    d.mip_level = mco_mip_level(sp->g1, sp->g2, b->mip_offset);
                    uint32_t t[2];
                    mco_texel(sp->uv, d.mip_level, t);
                    d.texel_x = t[0];
                    d.texel_y = t[1];
                }
                float hit[3];
                if (mco_cache_lookup(b->cache, &d, hit)) {
                    stack[top++] = (ins->flags & MCG_F_SCALAR_RESULT) ? val_s(hit[0])
                                                                      : val_c(hit[0], hit[1], hit[2]);
                    (*nodes_found)++;
                    pc += (size_t)ins->imm.i;
                } else {
                    pending[ins->bracket] = d;
                    pend_cell[ins->bracket] = mco_hash_cell(&d);
                    pend_check[ins->bracket] = mco_hash_check(&d);
                }
                break;
            }
            case MCG_OP_CACHE_STORE: { /* :350-357 */
                if (!b->cache) break;
                b->stores_attempted++;
                const Val t = stack[top - 1];
                const float rgb[3] = {t.x, t.y, t.z};
                if (b->deferred) {
                    PendingStore ps = {pend_cell[ins->bracket], pend_check[ins->bracket],
                                       mco_encode(rgb), b->key_base | ins->store_ord};
                    queue_push(b, ps);
                } else {
                    if (mco_cache_update(b->cache, &pending[ins->bracket], rgb, NULL, NULL) ==
                        MCG_INSERT_WON) {
                        b->stores_won++;
                    }
                }
                break;
            }
            case MCG_OP_END:
                return stack[--top];
        }
    }
}

static void read_sp(const float* p, ShadePt* sp) { memcpy(sp, p, sizeof(ShadePt)); }

static int cmp_store(const void* a, const void* b);
static void apply_queue(mco_cache* cache, Binding* b);

static void execute_points(const mcg_flat_scene* s, uint32_t slot, const float* sp, size_t n,
                           mco_cache* cache, int mip_offset, int deferred, float* values,
                           uint32_t* nodes, uint32_t* instrs) {
    Binding b;
    memset(&b, 0, sizeof(b));
    b.cache = cache;
    b.mip_offset = mip_offset;
    b.deferred = deferred;
    for (size_t i = 0; i < n; ++i) {
        ShadePt pt;
        read_sp(sp + 15 * i, &pt);
        uint32_t nf = 0;
        const uint64_t before = b.instructions;
        b.key_base = (uint32_t)i << 6;
        const Val v = execute(s, slot, &pt, &b, &nf);
        values[4 * i] = v.x;
        values[4 * i + 1] = v.y;
        values[4 * i + 2] = v.z;
        uint32_t tag = v.scalar ? 1u : 0u;
        memcpy(values + 4 * i + 3, &tag, 4);
        nodes[i] = nf;
        instrs[i] = (uint32_t)(b.instructions - before);
    }
    if (deferred) apply_queue(cache, &b);
    free(b.queue);
}

void mco_execute_batch(const mcg_flat_scene* s, uint32_t slot, const float* sp, size_t n,
                       mco_cache* cache, int mip_offset, float* values, uint32_t* nodes,
                       uint32_t* instrs) {
    execute_points(s, slot, sp, n, cache, mip_offset, 0, values, nodes, instrs);
}

void mco_execute_batch_deferred(const mcg_flat_scene* s, uint32_t slot, const float* sp, size_t n,
                                mco_cache* cache, int mip_offset, float* values, uint32_t* nodes,
                                uint32_t* instrs) {
    execute_points(s, slot, sp, n, cache, mip_offset, cache != NULL, values, nodes, instrs);
}

/* ------------------------------------------------------------ scene.cpp BVH */

typedef struct { V3 origin, dir; } Ray;

typedef struct {
    float t;
    uint32_t prim;
    float b1, b2;
} Hit;

/* ray_aabb: src/scene.cpp:42-56 */
static int ray_aabb(const Ray* r, const float lo[3], const float hi[3], float tmin, float tmax) {
    const float inv[3] = {1.0f / r->dir.x, 1.0f / r->dir.y, 1.0f / r->dir.z};
    const float o[3] = {r->origin.x, r->origin.y, r->origin.z};
    for (int a = 0; a < 3; ++a) {
        float t0 = (lo[a] - o[a]) * inv[a];
        float t1 = (hi[a] - o[a]) * inv[a];
        if (inv[a] < 0.0f) { const float tmp = t0; t0 = t1; t1 = tmp; }
        tmin = fmaxf(tmin, t0);
        tmax = fminf(tmax, t1);
        if (tmax < tmin) return 0;
    }
    return 1;
}

/* ray_triangle: src/scene.cpp:58-78 (e1, e2 precomputed as p1-p0, p2-p0) */
static int ray_tri(const Ray* r, const float* g, float tmin, float tmax, float* t, float* b1,
                   float* b2) {
    const V3 p0 = v3_load(g), e1 = v3_load(g + 4), e2 = v3_load(g + 8);
    const V3 pvec = v3_cross(r->dir, e2);
    const float det = v3_dot(e1, pvec);
    if (fabsf(det) < 1e-12f) return 0;
    const float inv_det = 1.0f / det;
    const V3 tvec = v3_sub(r->origin, p0);
    const float u = v3_dot(tvec, pvec) * inv_det;
    if (u < 0.0f || u > 1.0f) return 0;
    const V3 qvec = v3_cross(tvec, e1);
    const float v = v3_dot(r->dir, qvec) * inv_det;
    if (v < 0.0f || u + v > 1.0f) return 0;
    const float ht = v3_dot(e2, qvec) * inv_det;
    if (ht <= tmin || ht >= tmax) return 0;
    *t = ht;
    *b1 = u;
    *b2 = v;
    return 1;
}

/* ray_sphere: src/scene.cpp:80-94 */
static int ray_sphere(const Ray* r, const float* g, float tmin, float tmax, float* t) {
    const V3 c = v3_load(g);
    const float radius = g[3];
    const V3 oc = v3_sub(r->origin, c);
    const float b = v3_dot(oc, r->dir);
    const float cc = v3_dot(oc, oc) - radius * radius;
    const float disc = b * b - cc;
    if (disc < 0.0f) return 0;
    const float sq = sqrtf(disc);
    float root = -b - sq;
    if (root <= tmin || root >= tmax) {
        root = -b + sq;
        if (root <= tmin || root >= tmax) return 0;
    }
    *t = root;
    return 1;
}

static int prim_hit(const mcg_flat_scene* s, uint32_t i, const Ray* r, float tmin, float tmax,
                    Hit* h) {
    const float* g = s->prim_geom + 12 * (size_t)i;
    float t, b1 = 0, b2 = 0;
    if (s->prim_info[i] & MCG_PRIM_SPHERE) {
        if (!ray_sphere(r, g, tmin, tmax, &t)) return 0;
    } else {
        if (!ray_tri(r, g, tmin, tmax, &t, &b1, &b2)) return 0;
    }
    h->t = t;
    h->prim = i;
    h->b1 = b1;
    h->b2 = b2;
    return 1;
}

/* Scene::intersect: src/scene.cpp:252-278 (DFS, left pushed then right) */
static int intersect(const mcg_flat_scene* s, const Ray* r, float tmin, float tmax, Hit* out) {
    if (s->n_nodes == 0) return 0;
    int found = 0;
    float closest = tmax;
    int32_t stack[64];
    int top = 0;
    stack[top++] = 0;
    while (top > 0) {
        const mcg_bvh_node* nd = &s->nodes[stack[--top]];
        if (!ray_aabb(r, nd->lo, nd->hi, tmin, closest)) continue;
        if (nd->a < 0) {
            const uint32_t first = (uint32_t)~nd->a, count = (uint32_t)nd->b;
            for (uint32_t i = first; i < first + count; ++i) {
                Hit h;
                if (prim_hit(s, i, r, tmin, closest, &h)) {
                    closest = h.t;
                    *out = h;
                    found = 1;
                }
            }
        } else {
            stack[top++] = nd->a;
            stack[top++] = nd->b;
        }
    }
    return found;
}

/* Scene::occluded: src/scene.cpp:280-298 */
static int occluded(const mcg_flat_scene* s, const Ray* r, float tmin, float tmax) {
    if (s->n_nodes == 0) return 0;
    int32_t stack[64];
    int top = 0;
    stack[top++] = 0;
    while (top > 0) {
        const mcg_bvh_node* nd = &s->nodes[stack[--top]];
        if (!ray_aabb(r, nd->lo, nd->hi, tmin, tmax)) continue;
        if (nd->a < 0) {
            const uint32_t first = (uint32_t)~nd->a, count = (uint32_t)nd->b;
            for (uint32_t i = first; i < first + count; ++i) {
                Hit h;
                if (prim_hit(s, i, r, tmin, tmax, &h)) return 1;
            }
        } else {
            stack[top++] = nd->a;
            stack[top++] = nd->b;
        }
    }
    return 0;
}

typedef struct {
    V3 position, normal;
    V2 uv;
    V3 e1, e2;
    V2 duv1, duv2;
    uint32_t slot;
} Surface;

/* Hit record construction: src/scene.cpp:211-247 */
static void surface(const mcg_flat_scene* s, const Ray* r, const Hit* h, Surface* o) {
    const float* g = s->prim_geom + 12 * (size_t)h->prim;
    const uint32_t info = s->prim_info[h->prim];
    o->position = v3_add(r->origin, v3_mul(r->dir, h->t));
    o->slot = info & ~MCG_PRIM_SPHERE;
    if (!(info & MCG_PRIM_SPHERE)) {
        const V3 e1 = v3_load(g + 4), e2 = v3_load(g + 8);
        V3 n = v3_norm(v3_cross(e1, e2));
        if (v3_dot(n, r->dir) > 0.0f) { n.x = -n.x; n.y = -n.y; n.z = -n.z; }
        o->normal = n;
        const float* uv = s->prim_uv + 6 * (size_t)h->prim;
        const float w0 = 1.0f - h->b1 - h->b2;
        o->uv.x = uv[0] * w0 + uv[2] * h->b1 + uv[4] * h->b2;
        o->uv.y = uv[1] * w0 + uv[3] * h->b1 + uv[5] * h->b2;
        o->e1 = e1;
        o->e2 = e2;
        o->duv1.x = uv[2] - uv[0];
        o->duv1.y = uv[3] - uv[1];
        o->duv2.x = uv[4] - uv[0];
        o->duv2.y = uv[5] - uv[1];
        return;
    }
    /* sphere: scene.cpp:227-246; atan2f/acosf via mc_detmath.h (as the device) */
    const float kPi = 3.14159265358979323846f;
    const V3 c = v3_load(g);
    const float radius = g[3];
    const V3 m = v3_norm(v3_sub(o->position, c));
    V3 n = m;
    if (v3_dot(n, r->dir) > 0.0f) { n.x = -n.x; n.y = -n.y; n.z = -n.z; }
    o->normal = n;
    o->uv.x = 0.5f + mc_atan2f(m.z, m.x) / (2.0f * kPi);
    o->uv.y = mc_acosf(fminf(fmaxf(m.y, -1.0f), 1.0f)) / kPi;
    const float sin_t = sqrtf(fmaxf(0.0f, 1.0f - m.y * m.y));
    V3 du, dv;
    if (sin_t > 1e-6f) {
        V3 a = {-m.z, 0.0f, m.x};
        du = v3_mul(a, 2.0f * kPi * radius);
        const float cphi = m.x / sin_t, sphi = m.z / sin_t;
        V3 bq = {m.y * cphi, -sin_t, m.y * sphi};
        dv = v3_mul(bq, kPi * radius);
    } else {
        V3 a = {1, 0, 0}, bq = {0, 0, 1};
        du = v3_mul(a, 2.0f * kPi * radius);
        dv = v3_mul(bq, kPi * radius);
    }
    o->e1 = du;
    o->e2 = dv;
    o->duv1.x = 1.0f; o->duv1.y = 0.0f;
    o->duv2.x = 0.0f; o->duv2.y = 1.0f;
}

void mco_intersect_batch(const mcg_flat_scene* s, const float* rays, size_t n, float t_min,
                         float t_max, float* out) {
    for (size_t i = 0; i < n; ++i) {
        Ray r = {v3_load(rays + 6 * i), v3_load(rays + 6 * i + 3)};
        float* o = out + 24 * i;
        memset(o, 0, 24 * sizeof(float));
        Hit h;
        if (!intersect(s, &r, t_min, t_max, &h)) continue;
        Surface sf;
        surface(s, &r, &h, &sf);
        const float vals[21] = {1.0f, h.t, sf.position.x, sf.position.y, sf.position.z,
                                sf.normal.x, sf.normal.y, sf.normal.z, sf.uv.x, sf.uv.y,
                                (float)sf.slot, sf.e1.x, sf.e1.y, sf.e1.z, sf.e2.x, sf.e2.y,
                                sf.e2.z, sf.duv1.x, sf.duv1.y, sf.duv2.x, sf.duv2.y};
        memcpy(o, vals, sizeof(vals));
    }
}

void mco_occluded_batch(const mcg_flat_scene* s, const float* rays, size_t n, float t_min,
                        const float* t_max, uint8_t* out) {
    for (size_t i = 0; i < n; ++i) {
        Ray r = {v3_load(rays + 6 * i), v3_load(rays + 6 * i + 3)};
        out[i] = (uint8_t)occluded(s, &r, t_min, t_max[i]);
    }
}

/* --------------------------------------------------- render() (restated) */

#define K_TMIN 1e-4f
#define K_EPS 1e-4f
#define K_INV_PI 0.318309886183790671538f
#define K_TWO_PI 6.28318530717958647692f

void mco_camera_setup(const mcg_flat_scene* s, int w, int h, float out[12]) {
    const V3 pos = v3_load(s->cam_position);
    const V3 fwd = v3_norm(v3_sub(v3_load(s->cam_look_at), pos));
    const V3 right = v3_norm(v3_cross(fwd, v3_load(s->cam_up)));
    const V3 up = v3_cross(right, fwd);
    const float vfov = s->cam_vfov_deg * (3.14159265358979323846f / 180.0f);
    const float vals[12] = {fwd.x, fwd.y, fwd.z, right.x, right.y, right.z, up.x, up.y, up.z,
                            tanf(vfov * 0.5f), (float)w / (float)h,
                            /* cone_for_camera: src/raycone.cpp:8-13 */
                            atanf(2.0f * tanf(vfov * 0.5f) / (float)h)};
    memcpy(out, vals, sizeof(vals));
}

typedef struct {
    Ray ray;
    float cone_w, cone_s;
    V3 thr, L;
    uint32_t nodes;
    int alive;
} Path;

static uint32_t dim_rect(int b, int j, int k) { return 2u + 64u * (uint32_t)b + 2u * (uint32_t)j + (uint32_t)k; }
static uint32_t dim_bounce(int b, int k) { return 2u + 64u * (uint32_t)b + 62u + (uint32_t)k; }

static void path_start(const float cam[12], const float* cam_pos, int x, int y, int w, int h,
                       Rng rng, Path* p) {
    const float jx = rng_sample(rng, 0), jy = rng_sample(rng, 1);
    const float sx = (((float)x + jx) / (float)w) * 2.0f - 1.0f;
    const float sy = 1.0f - (((float)y + jy) / (float)h) * 2.0f;
    const float a = (sx * cam[9]) * cam[10];
    const float bq = sy * cam[9];
    const V3 fwd = v3_load(cam), right = v3_load(cam + 3), up = v3_load(cam + 6);
    const V3 d = v3_add(v3_add(fwd, v3_mul(right, a)), v3_mul(up, bq));
    memset(p, 0, sizeof(*p));
    p->ray.origin = v3_load(cam_pos);
    p->ray.dir = v3_norm(d);
    p->cone_w = 0.0f;
    p->cone_s = cam[11];
    p->thr.x = p->thr.y = p->thr.z = 1.0f;
    p->alive = 1;
}

static void add_light(Path* p, V3 tf, V3 emit, float w) {
    p->L.x = p->L.x + tf.x * (emit.x * w);
    p->L.y = p->L.y + tf.y * (emit.y * w);
    p->L.z = p->L.z + tf.z * (emit.z * w);
}

/* One path vertex. */
static void path_vertex(const mcg_flat_scene* s, const mco_render_params* rp, Binding* bind,
                        Rng rng, int b, Path* p, uint64_t* shading_points) {
    Hit h;
    if (!intersect(s, &p->ray, K_TMIN, INFINITY, &h)) {
        const V3 env = v3_load(s->env);
        p->L = v3_add(p->L, v3_hadamard(p->thr, env));
        p->alive = 0;
        return;
    }
    Surface sf;
    surface(s, &p->ray, &h, &sf);
    p->cone_w += h.t * p->cone_s; /* propagate: raycone.cpp:15-18 */
    V2 g1, g2;
    footprint(p->cone_w, p->ray.dir, sf.normal, sf.e1, sf.e2, sf.duv1, sf.duv2, &g1, &g2);
    ShadePt sp;
    sp.pos[0] = sf.position.x; sp.pos[1] = sf.position.y; sp.pos[2] = sf.position.z;
    sp.nrm[0] = sf.normal.x; sp.nrm[1] = sf.normal.y; sp.nrm[2] = sf.normal.z;
    sp.inc[0] = p->ray.dir.x; sp.inc[1] = p->ray.dir.y; sp.inc[2] = p->ray.dir.z;
    sp.uv[0] = sf.uv.x; sp.uv[1] = sf.uv.y;
    sp.g1[0] = g1.x; sp.g1[1] = g1.y; sp.g2[0] = g2.x; sp.g2[1] = g2.y;
    uint32_t nf = 0;
    const Val v = execute(s, sf.slot, &sp, bind, &nf);
    (*shading_points)++;
    p->nodes += nf;
    const V3 alb = {fminf(fmaxf(v.x, 0.0f), 1.0f), fminf(fmaxf(v.y, 0.0f), 1.0f),
                    fminf(fmaxf(v.z, 0.0f), 1.0f)};
    const V3 f = v3_mul(alb, K_INV_PI);
    const V3 tf = v3_hadamard(p->thr, f);
    const V3 n = sf.normal;
    const V3 o = v3_add(sf.position, v3_mul(n, K_EPS));
    for (uint32_t li = 0; li < s->n_point_lights; ++li) {
        const mcg_point_light* l = &s->point_lights[li];
        const V3 toL = v3_sub(v3_load(l->position), o);
        const float d2 = v3_dot(toL, toL);
        const float dist = sqrtf(d2);
        const V3 wi = v3_mul(toL, 1.0f / dist);
        const float cs = v3_dot(n, wi);
        Ray sr = {o, wi};
        if (cs > 0.0f && !occluded(s, &sr, K_TMIN, dist)) add_light(p, tf, v3_load(l->intensity), cs / d2);
    }
    for (uint32_t j = 0; j < s->n_rect_lights; ++j) {
        const mcg_rect_light* l = &s->rect_lights[j];
        const float u = rng_sample(rng, dim_rect(b, (int)j, 0));
        const float vv = rng_sample(rng, dim_rect(b, (int)j, 1));
        const V3 eu = v3_load(l->edge_u), ev = v3_load(l->edge_v);
        const V3 pl = v3_add(v3_add(v3_load(l->corner), v3_mul(eu, u)), v3_mul(ev, vv));
        const V3 nl = v3_cross(eu, ev);
        const float area = v3_len(nl);
        const V3 toL = v3_sub(pl, o);
        const float d2 = v3_dot(toL, toL);
        const float dist = sqrtf(d2);
        const V3 wi = v3_mul(toL, 1.0f / dist);
        const float cs = v3_dot(n, wi);
        const float cl = fabsf(v3_dot(nl, wi)) / area;
        Ray sr = {o, wi};
        if (cs > 0.0f && cl > 0.0f && !occluded(s, &sr, K_TMIN, dist)) {
            add_light(p, tf, v3_load(l->radiance), ((cs * cl) * area) / d2);
        }
    }
    if (b == rp->max_bounces) {
        p->alive = 0;
        return;
    }
    const float r1 = rng_sample(rng, dim_bounce(b, 0));
    const float r2 = rng_sample(rng, dim_bounce(b, 1));
    float sphi, cphi;
    mc_sincosf(r1 * K_TWO_PI, &sphi, &cphi);
    const float r = sqrtf(r2);
    const float lx = r * cphi, ly = r * sphi;
    const float lz = sqrtf(fmaxf(0.0f, 1.0f - r2));
    const float sign = copysignf(1.0f, n.z);
    const float a = -1.0f / (sign + n.z);
    const float bb = (n.x * n.y) * a;
    const V3 t = {1.0f + ((sign * n.x) * n.x) * a, sign * bb, -sign * n.x};
    const V3 bt = {bb, sign + ((n.y * n.y) * a), -n.y};
    const V3 nd = v3_norm(v3_add(v3_add(v3_mul(t, lx), v3_mul(bt, ly)), v3_mul(n, lz)));
    p->thr = v3_hadamard(p->thr, alb);
    p->cone_s += rp->diffuse_spread; /* widen: raycone.cpp:20-23 */
    p->ray.origin = o;
    p->ray.dir = nd;
}

static int tile_mine(const mco_render_params* p, int tile, int n_tiles) {
    if (p->shard_count <= 1) return 1;
    if (p->shard_mode == 0) return tile % p->shard_count == p->shard_rank;
    const int lo = (int)((int64_t)n_tiles * p->shard_rank / p->shard_count);
    const int hi = (int)((int64_t)n_tiles * (p->shard_rank + 1) / p->shard_count);
    return tile >= lo && tile < hi;
}

static int cmp_store(const void* a, const void* b) {
    const PendingStore* x = (const PendingStore*)a;
    const PendingStore* y = (const PendingStore*)b;
    return x->key < y->key ? -1 : (x->key > y->key ? 1 : 0);
}

/* Epoch end: the queued stores, in (sample, pixel, store ordinal) order, with
 * update() semantics (the deterministic-insert rule). */
static void apply_queue(mco_cache* cache, Binding* b) {
    if (!b->queue_len) return;
    qsort(b->queue, b->queue_len, sizeof(PendingStore), cmp_store);
    for (size_t q = 0; q < b->queue_len; ++q) {
        const PendingStore* ps = &b->queue[q];
        if (cache_update_hashed(cache, ps->cell_hash, ps->check, ps->payload, NULL, NULL) ==
            MCG_INSERT_WON) {
            b->stores_won++;
        }
    }
    b->queue_len = 0;
}

int mco_render(const mcg_flat_scene* s, const mco_render_params* p, mco_cache* external_cache,
               double* radiance, double* nodes_found, uint32_t* samples,
               uint64_t* hits_per_sample, mco_render_stats* stats) {
    if (p->mode != 0 && p->mode != 1 && p->mode != 3) return 1;
    const int w = p->width ? p->width : s->cam_width;
    const int h = p->height ? p->height : s->cam_height;
    float cam[12];
    mco_camera_setup(s, w, h, cam);
    mco_cache* cache = NULL;
    mco_cache* own = NULL;
    if (p->mode != 0) {
        cache = external_cache;
        if (!cache) cache = own = mco_cache_new(p->n_cells, p->n_entries);
        if (!cache) return 1;
        cache->lookups = cache->hits = cache->won = cache->lost_full = 0;
    }
    Binding bind;
    memset(&bind, 0, sizeof(bind));
    bind.cache = cache;
    bind.mip_offset = p->mip_offset;
    bind.deferred = p->mode == 3;

    const int ts = p->tile_size > 0 ? p->tile_size : 16;
    const int tiles_x = (w + ts - 1) / ts, tiles_y = (h + ts - 1) / ts;
    uint32_t* pix = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)w * h);
    size_t np = 0;
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x)
            if (tile_mine(p, (y / ts) * tiles_x + x / ts, tiles_x * tiles_y)) pix[np++] = (uint32_t)(y * w + x);
    const int k = p->samples_per_pass > 0 ? (p->samples_per_pass < p->spp ? p->samples_per_pass : p->spp) : 1;
    const uint32_t wh = (uint32_t)w * (uint32_t)h;
    Path* st = (Path*)calloc(np * (size_t)k + 1, sizeof(Path));
    struct timespec t0, t1;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    uint64_t shading = 0;
    for (int start = 0; start < p->spp; start += k) {
        const int kk = (p->spp - start) < k ? (p->spp - start) : k;
        for (int j = 0; j < kk; ++j) {
            const uint32_t sidx = p->first_sample + (uint32_t)(start + j);
            for (size_t q = 0; q < np; ++q) {
                path_start(cam, s->cam_position, (int)(pix[q] % (uint32_t)w), (int)(pix[q] / (uint32_t)w),
                           w, h, rng_make(p->rng_seed, pix[q], sidx), &st[(size_t)j * np + q]);
            }
        }
        for (int b = 0; b <= p->max_bounces; ++b) {
            /* One epoch: every path of this pass at bounce b, in (sample, pixel) order. */
            for (int j = 0; j < kk; ++j) {
                const uint32_t sidx = p->first_sample + (uint32_t)(start + j);
                for (size_t q = 0; q < np; ++q) {
                    Path* ps = &st[(size_t)j * np + q];
                    if (!ps->alive) continue;
                    bind.key_base = ((uint32_t)j * wh + pix[q]) << 6;
                    path_vertex(s, p, &bind, rng_make(p->rng_seed, pix[q], sidx), b, ps, &shading);
                }
            }
            if (bind.deferred) apply_queue(cache, &bind);
        }
        for (size_t q = 0; q < np; ++q) {
            for (int j = 0; j < kk; ++j) {
                const Path* ps = &st[(size_t)j * np + q];
                const uint32_t px = pix[q];
                radiance[3 * (size_t)px] += ps->L.x;
                radiance[3 * (size_t)px + 1] += ps->L.y;
                radiance[3 * (size_t)px + 2] += ps->L.z;
                nodes_found[px] += ps->nodes;
                samples[px] += 1;
                if (hits_per_sample) hits_per_sample[start + j] += ps->nodes;
            }
        }
    }
    clock_gettime(CLOCK_MONOTONIC, &t1);
    if (stats) {
        memset(stats, 0, sizeof(*stats));
        stats->wall_time_s = (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
        if (cache) {
            stats->lookups = cache->lookups;
            stats->hits = cache->hits;
            stats->inserts_won = cache->won;
            stats->inserts_lost_full = cache->lost_full;
        }
        stats->stores_attempted = bind.stores_attempted;
        stats->stores_won = bind.stores_won;
        stats->instructions_executed = bind.instructions;
        stats->paths = (uint64_t)np * (uint64_t)p->spp;
        stats->shading_points = shading;
    }
    free(bind.queue);
    free(st);
    free(pix);
    mco_cache_free(own);
    return 0;
}

/* ------------------------------------------------------------ batch glue */

void mco_hash_batch(const mcg_descriptor* d, size_t n, uint64_t* cell, uint32_t* check) {
    for (size_t i = 0; i < n; ++i) {
        cell[i] = mco_hash_cell(&d[i]);
        check[i] = mco_hash_check(&d[i]);
    }
}
void mco_encode_batch(const float* rgb, size_t n, uint32_t* out) {
    for (size_t i = 0; i < n; ++i) out[i] = mco_encode(rgb + 3 * i);
}
void mco_decode_batch(const uint32_t* in, size_t n, float* rgb) {
    for (size_t i = 0; i < n; ++i) mco_decode(in[i], rgb + 3 * i);
}
void mco_mip_texel_batch(const float* uv, const float* g1, const float* g2, size_t n, int off,
                         uint8_t* mip, uint32_t* txy) {
    for (size_t i = 0; i < n; ++i) {
        mip[i] = mco_mip_level(g1 + 2 * i, g2 + 2 * i, off);
        mco_texel(uv + 2 * i, mip[i], txy + 2 * i);
    }
}
void mco_footprint_batch(const float* in, size_t n, float* out) {
    for (size_t i = 0; i < n; ++i) mco_footprint(in + 17 * i, out + 4 * i);
}
void mco_fbm_batch(const int32_t* octaves, const float* fp, const float* uv, size_t n, float* out) {
    for (size_t i = 0; i < n; ++i) {
        mcg_noise p = {octaves[i], fp[3 * i], fp[3 * i + 1], fp[3 * i + 2]};
        out[i] = mco_fbm(&p, uv[2 * i], uv[2 * i + 1]);
    }
}
void mco_sin_wave_batch(const float* x, size_t n, float* out) {
    for (size_t i = 0; i < n; ++i) out[i] = mco_sin_wave(x[i]);
}
/* sphere uv's atan2f / acosf (mc_detmath.h) */
void mco_atan2f_batch(const float* y, const float* x, size_t n, float* out) {
    for (size_t i = 0; i < n; ++i) out[i] = mc_atan2f(y[i], x[i]);
}
void mco_acosf_batch(const float* x, size_t n, float* out) {
    for (size_t i = 0; i < n; ++i) out[i] = mc_acosf(x[i]);
}
void mco_power_batch(const float* x, const float* y, size_t n, float* out) {
    for (size_t i = 0; i < n; ++i) out[i] = mco_power(x[i], y[i]);
}

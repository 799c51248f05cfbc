// Device restatement of the reference's per-sample arithmetic. Every function
// evaluates the same IEEE operations in the same order as the reference
// (paths relative to /root/reference/proj/core); the library is compiled
// with --fmad=false so no multiply-add is ever contracted, matching the
// reference's -ffp-contract=off (proj/CMakeLists.txt:16). Bit-equality with
// the host is a parity test (tests/test_gpu_parity.py).
#pragma once

#include <cstdint>
#include <cstdio>

#include "../../include/mcg.h"

namespace mcgd {

// Checked builds (-DMCG_CHECKS=1; profiles/scripts/checked.sh): device-side
// bounds checks on every index the hot path computes -- the stand-in for
// compute-sanitizer, which this GPU pool does not allow. A failed check
// prints where and traps, so the launch (and the test driving it) fails.
#ifndef MCG_CHECKS
#define MCG_CHECKS 0
#endif
#if MCG_CHECKS
#define MCG_CHECK(cond)                                                                        \
    do {                                                                                       \
        if (!(cond)) {                                                                         \
            printf("MCG_CHECK failed: %s at %s:%d (block %d thread %d)\n", #cond, __FILE__,    \
                   __LINE__, static_cast<int>(blockIdx.x), static_cast<int>(threadIdx.x));     \
            __trap();                                                                          \
        }                                                                                      \
    } while (0)
#else
#define MCG_CHECK(cond) \
    do {                \
    } while (0)
#endif

constexpr int kMaxMip = 24;                       // raycone.hpp:18
constexpr float kTwoPi = 6.28318530717958647692f; // value.hpp:126

// ---------------------------------------------------------------- rng.hpp
#ifndef MCG_MIX_IMAD
#define MCG_MIX_IMAD 0
#endif
#if MCG_MIX_IMAD
// (experiment, off: probe lookups 40.4 vs 43.3 G/s -- more instructions in
// total) x ^ (x >> s) on 32-bit halves with the right shifts done as multiply-highs
// (IMAD.HI on the FMA pipe instead of SHF on the ALU pipe, which the hashing
// kernels saturate); integer arithmetic, so the result is the same word.
__device__ __forceinline__ uint64_t xorshr(uint64_t x, uint32_t s) {
    const uint32_t lo = static_cast<uint32_t>(x), hi = static_cast<uint32_t>(x >> 32);
    uint32_t m;   // 2^(32 - s), opaque to the compiler so it stays a multiply
    asm("mov.b32 %0, %1;" : "=r"(m) : "r"(1u << (32 - s)));
    const uint32_t lo_s = __umulhi(lo, m) | (hi * m), hi_s = __umulhi(hi, m);
    return (static_cast<uint64_t>(hi ^ hi_s) << 32) | (lo ^ lo_s);
}
__device__ __forceinline__ uint64_t mix64(uint64_t x) {  // rng.hpp:8-13
    x += 0x9e3779b97f4a7c15ull;
    x = xorshr(x, 30) * 0xbf58476d1ce4e5b9ull;
    x = xorshr(x, 27) * 0x94d049bb133111ebull;
    return xorshr(x, 31);
}
#else
__device__ __forceinline__ uint64_t mix64(uint64_t x) {  // rng.hpp:8-13
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
#endif

__device__ __forceinline__ uint64_t path_key(uint64_t seed, uint64_t pixel, uint64_t sample) {
    return mix64(seed ^ mix64(pixel ^ mix64(sample)));   // rng.hpp:20-21
}

__device__ __forceinline__ float path_sample(uint64_t key, uint32_t dim) {  // rng.hpp:24-27
    const uint64_t h = mix64(key + 0x632be59bd9b4e019ull * static_cast<uint64_t>(dim + 1));
    return static_cast<float>(h >> 40) * 0x1.0p-24f;
}

// -------------------------------------------------------------- cache.cpp
struct Desc {
    uint32_t mat, node, tx, ty;
    uint32_t mip;
};

// hash_descriptor (cache.cpp:21-30) for both seeds at once.
__device__ __forceinline__ void hash_desc(const Desc& d, uint64_t& cell_hash, uint32_t& check) {
    const uint64_t w0 = static_cast<uint64_t>(d.mat) | (static_cast<uint64_t>(d.node) << 32);
    const uint64_t w1 = static_cast<uint64_t>(d.tx) | (static_cast<uint64_t>(d.ty) << 32);
    const uint64_t w2 = d.mip;
    uint64_t a = 0x243f6a8885a308d3ull, b = 0x13198a2e03707344ull;
    a = mix64(a ^ w0);
    b = mix64(b ^ w0);
    a = mix64(a ^ w1);
    b = mix64(b ^ w1);
    a = mix64(a ^ w2);
    b = mix64(b ^ w2);
    cell_hash = a;
    const uint32_t c = static_cast<uint32_t>(b);
    check = c ? c : 1u;  // cache.cpp:36-39
}

// Exact h % n for a 64-bit h: q from the precomputed floor((2^64-1)/n),
// then at most two corrections (the estimate is low by <= 2).
__device__ __forceinline__ uint64_t fast_mod(uint64_t h, uint64_t n, uint64_t magic) {
    const uint64_t q = __umul64hi(h, magic);
    uint64_t r = h - q * n;
    if (r >= n) r -= n;
    if (r >= n) r -= n;
    return r;
}

// encode_value (cache.cpp:41-61), same double arithmetic.
__device__ __forceinline__ uint32_t encode_rgbe(float fr, float fg, float fb) {
    const double r = (isfinite(fr) && fr > 0.0f) ? static_cast<double>(fr) : 0.0;
    const double g = (isfinite(fg) && fg > 0.0f) ? static_cast<double>(fg) : 0.0;
    const double b = (isfinite(fb) && fb > 0.0f) ? static_cast<double>(fb) : 0.0;
    const double d = fmax(r, fmax(g, b));
    if (d <= 0.0) return 0u;
    int e = 0;
    frexp(d, &e);
    if (e < -127) return 0u;
    if (e > 127) e = 127;
    const double fac = ldexp(256.0, -e);
    uint32_t mr = static_cast<uint32_t>(r * fac), mg = static_cast<uint32_t>(g * fac),
             mb = static_cast<uint32_t>(b * fac);
    mr = mr > 255u ? 255u : mr;
    mg = mg > 255u ? 255u : mg;
    mb = mb > 255u ? 255u : mb;
    return (static_cast<uint32_t>(e + 128) << 24) | (mr << 16) | (mg << 8) | mb;
}

// decode_value (cache.cpp:63-71): (m + 0.5) * 2^(E-136) is exact in float
// (9 significant bits, E-136 >= -135 stays within the subnormal range), so
// the float path below equals the reference's double-then-round.
__device__ __forceinline__ float3 decode_rgbe(uint32_t p) {
    const uint32_t ex = p >> 24;
    if (ex == 0) return make_float3(0.0f, 0.0f, 0.0f);
    const int k = static_cast<int>(ex) - 136;
    return make_float3(ldexpf(static_cast<float>((p >> 16) & 255u) + 0.5f, k),
                       ldexpf(static_cast<float>((p >> 8) & 255u) + 0.5f, k),
                       ldexpf(static_cast<float>(p & 255u) + 0.5f, k));
}

// ------------------------------------------------------------ raycone.cpp
__device__ __forceinline__ float len2(float x, float y) { return sqrtf(x * x + y * y); }

// mip_level (raycone.cpp:67-73); floor(-log2 m) from the binary exponent:
// m = f 2^E, f in [0.5, 1): 1-E when f == 0.5, else -E.
__device__ __forceinline__ uint32_t mip_level(float g1x, float g1y, float g2x, float g2y,
                                              int offset) {
    const float m = fminf(len2(g1x, g1y), len2(g2x, g2y));
    if (!(m > 0.0f)) return kMaxMip;
    int32_t lv;
    if (isinf(m)) {
        // The reference converts floor(-inf) to INT_MIN (x86-64 cvttsd2si)
        // and adds the offset with wrap-around.
        lv = static_cast<int32_t>(0x80000000u + static_cast<uint32_t>(offset));
    } else {
        int e;
        const double f = frexp(static_cast<double>(m), &e);
        lv = (f == 0.5 ? 1 - e : -e) + offset;
    }
    return static_cast<uint32_t>(lv < 0 ? 0 : (lv > kMaxMip ? kMaxMip : lv));
}

// texel_indices (raycone.cpp:75-83)
__device__ __forceinline__ uint32_t texel_index(float t, uint32_t level) {
    const uint32_t res = 1u << level;
    const float w = t - floorf(t);
    const float s = w * static_cast<float>(res);
    const uint32_t i = (s != s) ? 0u : static_cast<uint32_t>(s);
    return i >= res ? res - 1 : i;
}

struct V3 {
    float x, y, z;
};
__device__ __forceinline__ V3 v3(float x, float y, float z) { return {x, y, z}; }
__device__ __forceinline__ V3 operator+(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ V3 operator-(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ V3 operator*(V3 a, float s) { return {a.x * s, a.y * s, a.z * s}; }
__device__ __forceinline__ float dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ V3 cross(V3 a, V3 b) {
    return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
__device__ __forceinline__ float length(V3 a) { return sqrtf(dot(a, a)); }
__device__ __forceinline__ V3 normalize(V3 a) {  // geom.hpp:34-37
    const float l = length(a);
    return l > 0.0f ? a * (1.0f / l) : V3{0.0f, 0.0f, 0.0f};
}

// world_to_uv (raycone.cpp:35-46)
__device__ __forceinline__ float2 world_to_uv(V3 a, V3 e1, V3 e2, float2 d1, float2 d2) {
    const float g11 = dot(e1, e1), g12 = dot(e1, e2), g22 = dot(e2, e2);
    const float det = g11 * g22 - g12 * g12;
    if (fabsf(det) < 1e-20f) return make_float2(0.0f, 0.0f);
    const float r1 = dot(a, e1), r2 = dot(a, e2);
    const float alpha = (r1 * g22 - r2 * g12) / det;
    const float beta = (r2 * g11 - r1 * g12) / det;
    return make_float2(d1.x * alpha + d2.x * beta, d1.y * alpha + d2.y * beta);
}

// footprint_gradients (raycone.cpp:50-65; any_tangent :28-31)
__device__ __forceinline__ void footprint(float width, V3 inc, V3 n, V3 e1, V3 e2, float2 d1,
                                          float2 d2, float2& g1, float2& g2) {
    const float cos_t = fmaxf(fabsf(dot(inc, n)), 1e-4f);
    const V3 proj = inc - n * dot(inc, n);
    const float plen = length(proj);
    V3 ax1;
    if (plen > 1e-6f) {
        ax1 = proj * (1.0f / plen);
    } else {
        const V3 axis = fabsf(n.x) < 0.9f ? V3{1.0f, 0.0f, 0.0f} : V3{0.0f, 1.0f, 0.0f};
        ax1 = normalize(cross(n, axis));
    }
    const V3 ax2 = normalize(cross(n, ax1));
    const float half_major = width / (2.0f * cos_t);
    const float half_minor = width * 0.5f;
    g1 = world_to_uv(ax1 * half_major, e1, e2, d1, d2);
    g2 = world_to_uv(ax2 * half_minor, e1, e2, d1, d2);
}

// -------------------------------------------------------------- noise.cpp
// Ken Perlin's permutation (noise.cpp:12-29); kernels stage it in shared
// memory because perlin2 indexes it divergently.
static __constant__ uint8_t kPermTable[256] = {
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

__device__ __forceinline__ void stage_perm(uint8_t* s_perm) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) s_perm[i] = kPermTable[i];
}

__device__ __forceinline__ float fade(float t) {
    return t * t * t * (t * (t * 6.0f - 15.0f) + 10.0f);
}
__device__ __forceinline__ float lerp(float a, float b, float t) { return a + (b - a) * t; }
// grad2 (noise.cpp): the 8 gradients as selects, not an 8-way switch (the
// hash is per lane, so a switch diverges inside the FBM loop). Same values
// bit for bit: x - y is x + (-y) in IEEE arithmetic, and +-dx / +-dy are
// returned unrounded as the switch returns them.
__device__ __forceinline__ float grad2(int h, float dx, float dy) {
    const float xs = (h & 1) ? -dx : dx;
    const float ys = (h & 2) ? -dy : dy;
    const float axis = (h & 2) ? ((h & 1) ? -dy : dy) : xs;   // h = 4, 5: +-dx; 6, 7: +-dy
    return (h & 4) ? axis : xs + ys;
}

// perlin2 (noise.cpp:53-75); perm is the 256-entry table staged in shared memory.
__device__ __forceinline__ float perlin2(float x, float y, const uint8_t* perm) {
    const float fx = floorf(x), fy = floorf(y);
    const int ix = static_cast<int>(fx), iy = static_cast<int>(fy);
    const float dx = x - fx, dy = y - fy;
    const float u = fade(dx), v = fade(dy);
    const int a = perm[ix & 255] + iy;
    const int b = perm[(ix + 1) & 255] + iy;
    const float n00 = grad2(perm[a & 255], dx, dy);
    const float n10 = grad2(perm[b & 255], dx - 1.0f, dy);
    const float n01 = grad2(perm[(a + 1) & 255], dx, dy - 1.0f);
    const float n11 = grad2(perm[(b + 1) & 255], dx - 1.0f, dy - 1.0f);
    const float n = lerp(lerp(n00, n10, u), lerp(n01, n11, u), v);
    return n * 1.41421356f;
}

// fbm2 (noise.cpp:77-91)
__device__ __forceinline__ float fbm2(const mcg_noise& p, float u, float v, const uint8_t* perm) {
    const int oct = p.octaves < 1 ? 1 : (p.octaves > 10 ? 10 : p.octaves);
    float sum = 0.0f, amp = 1.0f, norm = 0.0f, freq = p.frequency;
    for (int o = 0; o < oct; ++o) {
        sum += amp * perlin2(u * freq, v * freq, perm);
        norm += amp;
        amp *= p.gain;
        freq *= p.lacunarity;
    }
    const float n = norm > 0.0f ? sum / norm : 0.0f;
    return fminf(fmaxf(0.5f + 0.5f * n, 0.0f), 1.0f);
}

// ------------------------------------------------------------ texture.cpp
__device__ __forceinline__ float wrap_coord(float t, bool clamp) {
    return clamp ? fminf(fmaxf(t, 0.0f), 1.0f) : t - floorf(t);
}
__device__ __forceinline__ int wrap_index(int i, int n, bool clamp) {
    if (!clamp) {
        i %= n;
        return i < 0 ? i + n : i;
    }
    return i < 0 ? 0 : (i >= n ? n - 1 : i);
}

// sample_bilinear (texture.cpp:24-48): four 128-bit texel loads.
__device__ __forceinline__ float3 bilinear(const mcg_texture& t, const float4* texels, float uu,
                                           float vv, bool clamp) {
    const float u = wrap_coord(uu, clamp), v = wrap_coord(vv, clamp);
    const float x = u * static_cast<float>(t.width) - 0.5f;
    const float y = v * static_cast<float>(t.height) - 0.5f;
    const float fx = floorf(x), fy = floorf(y);
    const float tx = x - fx, ty = y - fy;
    const int x0 = wrap_index(static_cast<int>(fx), t.width, clamp);
    const int x1 = wrap_index(static_cast<int>(fx) + 1, t.width, clamp);
    const int y0 = wrap_index(static_cast<int>(fy), t.height, clamp);
    const int y1 = wrap_index(static_cast<int>(fy) + 1, t.height, clamp);
    const float4* px = texels + t.offset;
    MCG_CHECK(x0 >= 0 && x0 < t.width && x1 >= 0 && x1 < t.width && y0 >= 0 && y0 < t.height && y1 >= 0 &&
              y1 < t.height);
    const float4 c00 = __ldg(px + static_cast<size_t>(y0) * t.width + x0);
    const float4 c10 = __ldg(px + static_cast<size_t>(y0) * t.width + x1);
    const float4 c01 = __ldg(px + static_cast<size_t>(y1) * t.width + x0);
    const float4 c11 = __ldg(px + static_cast<size_t>(y1) * t.width + x1);
    const float wx = 1.0f - tx, wy = 1.0f - ty;
    const float tr = c00.x * wx + c10.x * tx, br = c01.x * wx + c11.x * tx;
    const float tg = c00.y * wx + c10.y * tx, bg = c01.y * wx + c11.y * tx;
    const float tb = c00.z * wx + c10.z * tx, bb = c01.z * wx + c11.z * tx;
    return make_float3(tr * wy + br * ty, tg * wy + bg * ty, tb * wy + bb * ty);
}

// checker (texture.cpp:50-54)
__device__ __forceinline__ float checker(float scale, float u, float v) {
    const int iu = static_cast<int>(floorf(u * scale));
    const int iv = static_cast<int>(floorf(v * scale));
    return ((iu + iv) & 1) == 0 ? 1.0f : 0.0f;
}

// ------------------------------------------------- deterministic sin / pow
// Double-precision routines rounded once to float; the CPU oracle evaluates
// the identical sequence. Replaces glibc sinf/powf at
// value.hpp:127 and :134.
__device__ __forceinline__ double sin_poly(double r) {
    const double z = r * r;
    double p = 1.0 / 355687428096000.0;
    p = p * z - 1.0 / 1307674368000.0;
    p = p * z + 1.0 / 6227020800.0;
    p = p * z - 1.0 / 39916800.0;
    p = p * z + 1.0 / 362880.0;
    p = p * z - 1.0 / 5040.0;
    p = p * z + 1.0 / 120.0;
    p = p * z - 1.0 / 6.0;
    return r + (r * z) * p;
}
__device__ __forceinline__ double cos_poly(double r) {
    const double z = r * r;
    double p = 1.0 / 6402373705728000.0;
    p = p * z - 1.0 / 20922789888000.0;
    p = p * z + 1.0 / 87178291200.0;
    p = p * z - 1.0 / 479001600.0;
    p = p * z + 1.0 / 3628800.0;
    p = p * z - 1.0 / 40320.0;
    p = p * z + 1.0 / 720.0;
    p = p * z - 1.0 / 24.0;
    p = p * z + 0.5;
    return 1.0 - z * p;
}
__device__ __forceinline__ void det_sincosf(float a, float& s_out, float& c_out) {
    const double x = static_cast<double>(a);
    if (!(x - x == 0.0)) {
        s_out = c_out = static_cast<float>(x - x);
        return;
    }
    const double k = rint(x * 6.36619772367581382433e-01);
    const double r = ((x - k * 1.57079632673412561417e+00) - k * 6.07710050630396597660e-11) -
                     k * 2.02226624879595063154e-21;
    const double sr = sin_poly(r), cr = cos_poly(r);
    const double kq = k - 4.0 * floor(k * 0.25);
    const int q = static_cast<int>(kq);
    double s, c;
    if (q == 0) { s = sr; c = cr; }
    else if (q == 1) { s = cr; c = -sr; }
    else if (q == 2) { s = -sr; c = -cr; }
    else { s = -cr; c = sr; }
    s_out = static_cast<float>(s);
    c_out = static_cast<float>(c);
}
__device__ __forceinline__ float det_sinf(float a) {
    float s, c;
    det_sincosf(a, s, c);
    return s;
}
__device__ __forceinline__ double log2_pos(double x) {
    int e;
    double m = frexp(x, &e);
    if (m < 0.70710678118654752440) {
        m = m * 2.0;
        e = e - 1;
    }
    const double t = (m - 1.0) / (m + 1.0);
    const double t2 = t * t;
    double p = 1.0 / 25.0;
    p = p * t2 + 1.0 / 23.0;
    p = p * t2 + 1.0 / 21.0;
    p = p * t2 + 1.0 / 19.0;
    p = p * t2 + 1.0 / 17.0;
    p = p * t2 + 1.0 / 15.0;
    p = p * t2 + 1.0 / 13.0;
    p = p * t2 + 1.0 / 11.0;
    p = p * t2 + 1.0 / 9.0;
    p = p * t2 + 1.0 / 7.0;
    p = p * t2 + 1.0 / 5.0;
    p = p * t2 + 1.0 / 3.0;
    p = p * t2 + 1.0;
    const double ln_m = 2.0 * (t * p);
    return static_cast<double>(e) + ln_m * 1.44269504088896340736;
}
__device__ __forceinline__ double exp2_det(double z) {
    if (z > 1100.0) return __longlong_as_double(0x7ff0000000000000ll);
    if (z < -1100.0) return 0.0;
    const double n = rint(z);
    const double f = (z - n) * 0.69314718055994530942;
    double p = 1.0 / 6402373705728000.0;
    p = p * f + 1.0 / 355687428096000.0;
    p = p * f + 1.0 / 20922789888000.0;
    p = p * f + 1.0 / 1307674368000.0;
    p = p * f + 1.0 / 87178291200.0;
    p = p * f + 1.0 / 6227020800.0;
    p = p * f + 1.0 / 479001600.0;
    p = p * f + 1.0 / 39916800.0;
    p = p * f + 1.0 / 3628800.0;
    p = p * f + 1.0 / 362880.0;
    p = p * f + 1.0 / 40320.0;
    p = p * f + 1.0 / 5040.0;
    p = p * f + 1.0 / 720.0;
    p = p * f + 1.0 / 120.0;
    p = p * f + 1.0 / 24.0;
    p = p * f + 1.0 / 6.0;
    p = p * f + 0.5;
    p = p * f + 1.0;
    p = p * f + 1.0;
    return ldexp(p, static_cast<int>(n));
}
__device__ __forceinline__ float det_powf_nonneg(float xf, float yf) {
    if (yf == 0.0f) return 1.0f;
    if (xf == 1.0f) return 1.0f;
    if (xf != xf || yf != yf) return xf + yf;
    const float inf = __int_as_float(0x7f800000);
    if (xf == 0.0f) return yf > 0.0f ? 0.0f : inf;
    if (isinf(xf)) return yf > 0.0f ? inf : 0.0f;
    if (isinf(yf)) {
        if (xf < 1.0f) return yf > 0.0f ? 0.0f : inf;
        return yf > 0.0f ? inf : 0.0f;
    }
    return static_cast<float>(exp2_det(static_cast<double>(yf) * log2_pos(static_cast<double>(xf))));
}

// atan2f / acosf of the sphere parameterization (scene.cpp:234-235): the
// same double-precision sequence as oracle/mc_detmath.h (mc_atan_unit,
// mc_atan2_d, mc_acosf), rounded once to float.
__device__ __forceinline__ double atan_unit(double t) {
    double base = 0.0;
    if (t > 0.41421356237309504880) {
        t = (t - 1.0) / (t + 1.0);
        base = 0.78539816339744830962;
    }
    const double h = t / (1.0 + sqrt(1.0 + t * t));
    const double z = h * h;
    double p = -1.0 / 23.0;
    p = p * z + 1.0 / 21.0;
    p = p * z - 1.0 / 19.0;
    p = p * z + 1.0 / 17.0;
    p = p * z - 1.0 / 15.0;
    p = p * z + 1.0 / 13.0;
    p = p * z - 1.0 / 11.0;
    p = p * z + 1.0 / 9.0;
    p = p * z - 1.0 / 7.0;
    p = p * z + 1.0 / 5.0;
    p = p * z - 1.0 / 3.0;
    return base + 2.0 * (h + (h * z) * p);
}
__device__ __forceinline__ double atan2_det(double y, double x) {
    if (x != x || y != y) return x + y;
    const double ax = fabs(x), ay = fabs(y);
    double a;
    if (ay == 0.0) a = 0.0;
    else if (isinf(ax) && isinf(ay)) a = 0.78539816339744830962;
    else if (ay <= ax) a = atan_unit(ay / ax);
    else a = 1.57079632679489661923 - atan_unit(ax / ay);
    if (signbit(x)) a = 3.14159265358979323846 - a;
    return copysign(a, y);
}
__device__ __forceinline__ float det_atan2f(float y, float x) {
    return static_cast<float>(atan2_det(static_cast<double>(y), static_cast<double>(x)));
}
__device__ __forceinline__ float det_acosf(float a) {
    const double x = static_cast<double>(a);
    if (x != x || fabs(x) > 1.0) return static_cast<float>((x - x) / (x - x));
    return static_cast<float>(atan2_det(sqrt((1.0 - x) * (1.0 + x)), x));
}

// sin_wave / power node kernels (value.hpp:125-137)
__device__ __forceinline__ float sin_wave(float x) { return 0.5f + 0.5f * det_sinf(x * kTwoPi); }
__device__ __forceinline__ float power(float x, float y) {
    const float r = det_powf_nonneg(fmaxf(x, 0.0f), y);
    return isfinite(r) ? r : 0.0f;
}

}  // namespace mcgd

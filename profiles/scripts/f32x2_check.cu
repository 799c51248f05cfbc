// Packed f32x2 vs scalar fp32: bit-compare add/sub/mul on random bit patterns.
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <vector>
#include <random>
__global__ void k(const float* a, const float* b, uint32_t* bad, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (2 * i + 1 >= n) return;
    float a0 = a[2 * i], a1 = a[2 * i + 1], b0 = b[2 * i], b1 = b[2 * i + 1];
    unsigned long long A = (unsigned long long)__float_as_uint(a1) << 32 | __float_as_uint(a0);
    unsigned long long B = (unsigned long long)__float_as_uint(b1) << 32 | __float_as_uint(b0);
    unsigned long long s, d, m;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(s) : "l"(A), "l"(B));
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(A), "l"(B));
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(m) : "l"(A), "l"(B));
    float s0 = __fadd_rn(a0, b0), s1 = __fadd_rn(a1, b1);
    float d0 = __fsub_rn(a0, b0), d1 = __fsub_rn(a1, b1);
    float m0 = __fmul_rn(a0, b0), m1 = __fmul_rn(a1, b1);
    if ((uint32_t)s != __float_as_uint(s0) || (uint32_t)(s >> 32) != __float_as_uint(s1)) atomicAdd(bad, 1);
    if ((uint32_t)d != __float_as_uint(d0) || (uint32_t)(d >> 32) != __float_as_uint(d1)) atomicAdd(bad + 1, 1);
    if ((uint32_t)m != __float_as_uint(m0) || (uint32_t)(m >> 32) != __float_as_uint(m1)) atomicAdd(bad + 2, 1);
}
int main() {
    const int n = 1 << 24;
    std::vector<float> a(n), b(n);
    std::mt19937 g(1);
    std::uniform_real_distribution<float> u(-10.f, 10.f);
    for (int i = 0; i < n; ++i) { a[i] = u(g); b[i] = u(g); }
    for (int i = 0; i < 1024; ++i) { uint32_t x = 0x00000100u + i; memcpy(&a[i], &x, 4); }  // denormals
    float *da, *db; uint32_t* dbad;
    cudaMalloc(&da, n * 4); cudaMalloc(&db, n * 4); cudaMalloc(&dbad, 12); cudaMemset(dbad, 0, 12);
    cudaMemcpy(da, a.data(), n * 4, cudaMemcpyHostToDevice); cudaMemcpy(db, b.data(), n * 4, cudaMemcpyHostToDevice);
    k<<<n / 2 / 256 + 1, 256>>>(da, db, dbad, n);
    uint32_t bad[3]; cudaMemcpy(bad, dbad, 12, cudaMemcpyDeviceToHost);
    printf("mismatches add %u sub %u mul %u of %d pairs\n", bad[0], bad[1], bad[2], n / 2);
    return 0;
}

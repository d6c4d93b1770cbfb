// Are the packed f32x2 multiply / add bit-identical to scalar RN ops? (W8A8 exact epilogue)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_f32x2 tools/ubench_f32x2.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void each(const float *a, const float *b, const float *c, int n, unsigned *bad) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (2 * i + 1 >= n) return;
    float x0 = a[2 * i], x1 = a[2 * i + 1], y0 = b[2 * i], y1 = b[2 * i + 1], z0 = c[2 * i], z1 = c[2 * i + 1];
    unsigned long long X = ((unsigned long long)__float_as_uint(x1) << 32) | __float_as_uint(x0);
    unsigned long long Y = ((unsigned long long)__float_as_uint(y1) << 32) | __float_as_uint(y0);
    unsigned long long Z = ((unsigned long long)__float_as_uint(z1) << 32) | __float_as_uint(z0);
    unsigned long long m, ad, f;
    asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(m) : "l"(X), "l"(Y));
    asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(ad) : "l"(X), "l"(Y));
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(f) : "l"(X), "l"(Y), "l"(Z));
    if ((unsigned)m != __float_as_uint(__fmul_rn(x0, y0)) || (unsigned)(m >> 32) != __float_as_uint(__fmul_rn(x1, y1))) atomicAdd(bad + 1, 1u);
    if ((unsigned)ad != __float_as_uint(__fadd_rn(x0, y0)) || (unsigned)(ad >> 32) != __float_as_uint(__fadd_rn(x1, y1))) atomicAdd(bad + 2, 1u);
    if ((unsigned)f != __float_as_uint(__fmaf_rn(x0, y0, z0)) || (unsigned)(f >> 32) != __float_as_uint(__fmaf_rn(x1, y1, z1))) atomicAdd(bad + 3, 1u);
}

__global__ void k(const float *a, const float *b, const float *c, int n, unsigned *bad) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (2 * i + 1 >= n) return;
    float x0 = a[2 * i], x1 = a[2 * i + 1], y0 = b[2 * i], y1 = b[2 * i + 1], z0 = c[2 * i], z1 = c[2 * i + 1];
    // scalar reference: (x*y)*z + c
    float s0 = __fadd_rn(__fmul_rn(__fmul_rn(x0, y0), z0), x1);
    float s1 = __fadd_rn(__fmul_rn(__fmul_rn(x1, y1), z1), x0);
    unsigned long long X = ((unsigned long long)__float_as_uint(x1) << 32) | __float_as_uint(x0);
    unsigned long long Y = ((unsigned long long)__float_as_uint(y1) << 32) | __float_as_uint(y0);
    unsigned long long Z = ((unsigned long long)__float_as_uint(z1) << 32) | __float_as_uint(z0);
    unsigned long long W = ((unsigned long long)__float_as_uint(x0) << 32) | __float_as_uint(x1);
    unsigned long long t, u, v;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(X), "l"(Y));
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(u) : "l"(t), "l"(Z));
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(v) : "l"(u), "l"(W));
    float p0 = __uint_as_float((unsigned)v), p1 = __uint_as_float((unsigned)(v >> 32));
    if (__float_as_uint(p0) != __float_as_uint(s0) || __float_as_uint(p1) != __float_as_uint(s1)) atomicAdd(bad, 1u);
}

int main() {
    const int n = 1 << 24;
    float *h = (float *)malloc(3 * n * sizeof(float));
    uint32_t s = 12345;
    for (int i = 0; i < 3 * n; i++) {
        s = s * 1664525u + 1013904223u;
        int e = (int)(s >> 27) - 16;
        float m = (float)((s >> 8) & 0xFFFF) / 65536.0f + 0.5f;
        h[i] = ((s & 1) ? -m : m) * ldexpf(1.0f, e);
    }
    float *d; unsigned *bad, hb[4] = {0, 0, 0, 0};
    cudaMalloc(&d, 3 * n * sizeof(float)); cudaMalloc(&bad, 16); cudaMemset(bad, 0, 16);
    cudaMemcpy(d, h, 3 * n * sizeof(float), cudaMemcpyHostToDevice);
    k<<<n / 2 / 256, 256>>>(d, d + n, d + 2 * n, n, bad);
    each<<<n / 2 / 256, 256>>>(d, d + n, d + 2 * n, n, bad);
    cudaMemcpy(hb, bad, 16, cudaMemcpyDeviceToHost);
    printf("pairs %d: chain mismatches %u; mul.f32x2 %u, add.f32x2 %u, fma.f32x2 %u (%s)\n", n / 2, hb[0], hb[1],
           hb[2], hb[3], cudaGetErrorString(cudaGetLastError()));
}

// Microbenchmark: tcgen05.ld (32x32b.x16) throughput per SM, 4 or 8 warps.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2512_16093_b200/csrc/ptx.cuh"
using namespace tb;
__global__ void __launch_bounds__(256, 1) k(int iters, int nwarps, unsigned long long *out, unsigned *sink) {
    __shared__ uint32_t taddr;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) ptx::tmem_alloc<256>(&taddr);
    ptx::tc_fence_before(); __syncthreads(); ptx::tc_fence_after();
    uint32_t acc = 0;
    unsigned long long t0 = clock64();
    if (warp < nwarps) {
        const uint32_t base = taddr + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 64;
        for (int it = 0; it < iters; it++) {
            uint32_t r[4][16];
#pragma unroll
            for (int q = 0; q < 4; q++) ptx::tmem_ld16(base + q * 16, r[q]);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int q = 0; q < 4; q++) acc += r[q][0] ^ r[q][15];
        }
    }
    __syncthreads();
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    if (acc == 0x12345) sink[0] = acc;
    ptx::tc_fence_before(); __syncthreads();
    if (warp == 0) ptx::tmem_dealloc<256>(taddr);
}
int main() {
    unsigned long long *d; unsigned *s; cudaMalloc(&d, 8 * 148); cudaMalloc(&s, 4);
    for (int nw : {1, 4, 8}) {
        int iters = 2000;
        k<<<148, 256>>>(iters, nw, d, s); cudaDeviceSynchronize();
        k<<<148, 256>>>(iters, nw, d, s); cudaDeviceSynchronize();
        unsigned long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        double bytes = (double)iters * nw * 32 * 64 * 4;   // per SM
        printf("warps %d: %llu cycles, %.1f B/clk/SM (%.1f cycles per 8KB warp-load of 64 cols)\n", nw, h, bytes / h,
               (double)h / iters);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}

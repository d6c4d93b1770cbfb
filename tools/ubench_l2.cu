// L2 -> SM bandwidth with TMA bulk loads (B200): every CTA streams 16 KB tiles
// from pseudo-random offsets of an L2-resident buffer through a 4-stage smem
// ring.  Reports aggregate TB/s for 1 and 2 CTAs per SM and two region sizes.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/ubench_l2 tools/ubench_l2.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2512_16093_b200/csrc/ptx.cuh"
using namespace tb;
constexpr int TILE = 16384, ST = 4;
__global__ void __launch_bounds__(32) k(const uint8_t *buf, size_t region_tiles, int iters, unsigned *sink) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t full[ST];
    if (threadIdx.x == 0) {
        for (int s = 0; s < ST; s++) ptx::mbar_init(&full[s], 1);
        ptx::fence_barrier_init();
    }
    __syncwarp();
    uint32_t x = blockIdx.x * 2654435761u + 12345u, acc = 0;
    if (threadIdx.x == 0) {
        for (int i = 0; i < iters + ST; i++) {
            const int s = i % ST;
            if (i >= ST) {
                ptx::mbar_wait(&full[s], ((i - ST) / ST) & 1);
                acc += smem[s * TILE + (i & 127)];
            }
            if (i < iters) {
                x = x * 1664525u + 1013904223u;
                const size_t t = x % region_tiles;
                ptx::mbar_arrive_expect_tx(&full[s], TILE);
                ptx::bulk_g2s(smem + s * TILE, buf + t * TILE, TILE, &full[s]);
            }
        }
    }
    if (acc == 0x12345678) sink[0] = acc;
}
int main() {
    uint8_t *buf;
    unsigned *sink;
    const size_t big = 1ull << 30;
    cudaMalloc(&buf, big);
    cudaMemset(buf, 1, big);
    cudaMalloc(&sink, 4);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, ST * TILE);
    for (size_t region : {32ull << 20, 64ull << 20, 1ull << 30}) {
        for (int per_sm : {1, 2, 4}) {
            const int grid = 148 * per_sm, iters = 2000;
            k<<<grid, 32, ST * TILE>>>(buf, region / TILE, 200, sink);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            k<<<grid, 32, ST * TILE>>>(buf, region / TILE, iters, sink);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("region %5zu MB, %d CTA/SM: %.2f TB/s\n", region >> 20, per_sm,
                   (double)grid * iters * TILE / (ms * 1e-3) / 1e12);
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}

// tcgen05 issue-queue depth: clock cycles a single thread spends issuing N
// M128 N128 K16 bf16 MMAs (64 clk each) back to back, without waiting.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2512_16093_b200/csrc/ptx.cuh"
using namespace tb;
__global__ void __launch_bounds__(128, 1) kq(int n, unsigned long long *out) {
    extern __shared__ uint8_t smd[];
    uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smd) + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t taddr;
    __shared__ uint64_t bar;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) ptx::tmem_alloc<512>(&taddr);
    if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_barrier_init(); }
    ptx::tc_fence_before(); __syncthreads(); ptx::tc_fence_after();
    if (warp == 0) {
        const uint64_t ad = ptx::sdesc_sw128(ptx::smem_u32(sm)), bd = ptx::sdesc_sw128(ptx::smem_u32(sm + 16384));
        const uint32_t id = ptx::idesc_bf16(128, 128);
        unsigned long long t0 = clock64(), t1 = 0;
        for (int i = 0; i < n; i++) {
            if (ptx::elect_one()) ptx::mma_f16(taddr + (i & 1) * 128, ad, bd, id, 1);
            __syncwarp();
            if (i == n - 1) t1 = clock64();
        }
        if (ptx::elect_one()) ptx::mma_commit(&bar);
        __syncwarp();
        ptx::mbar_wait(&bar, 0);
        unsigned long long t2 = clock64();
        if (threadIdx.x == 0) { out[2 * blockIdx.x] = t1 - t0; out[2 * blockIdx.x + 1] = t2 - t0; }
    }
    ptx::tc_fence_before(); __syncthreads();
    if (warp == 0) ptx::tmem_dealloc<512>(taddr);
}
int main() {
    unsigned long long *d, h[2];
    cudaMalloc(&d, 16 * 148);
    cudaFuncSetAttribute(kq, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
    for (int n : {1, 2, 3, 4, 6, 8, 12, 16, 24, 32, 48, 64}) {
        for (int rep = 0; rep < 2; rep++) { kq<<<148, 128, 40 * 1024>>>(n, d); cudaDeviceSynchronize(); }
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("N=%2d MMAs: issue %6llu clk, complete %6llu clk\n", n, h[0], h[1]);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}

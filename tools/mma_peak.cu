// mma_peak.cu -- measured dense tensor-core peak of this B200 (the roofline
// denominators of bench.py; VERDICT r01 "measure the real denominators").
//
// Every SM issues back-to-back tcgen05.mma from shared-memory operands (no
// loads, no epilogue): M128 N256 (cta_group::1, one CTA per SM) or M256 N256
// (cta_group::2, one CTA pair per two SMs), K = 32 bytes per instruction,
// two TMEM accumulators alternated so consecutive MMAs are independent.
// kind: 0 = kind::i8 (s32 D), 1 = kind::f16 bf16 (f32 D), 2 = kind::f8f6f4
// e4m3 (f32 D).  Work per launch = iters x M x N x K x 2 per CTA (pair).
// tools/mma_peak.py times launches with CUDA events (burst) and a
// seconds-long back-to-back loop (sustained), sampling NVML clocks.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -shared
//        -Xcompiler -fPIC -o tools/libmma_peak.so tools/mma_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2512_16093_b200/csrc/ptx.cuh"
using namespace tb;

namespace {

template <int KIND>
__host__ __device__ constexpr uint32_t idesc(int M, int N) {
    return KIND == 0 ? ptx::idesc_i8(M, N) : (KIND == 1 ? ptx::idesc_bf16(M, N) : ptx::idesc_e4m3(M, N));
}

template <int KIND, int CG>
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id) {
    if constexpr (CG == 1) {
        if constexpr (KIND == 0)
            asm volatile("tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, 1;" :: "r"(d), "l"(a), "l"(b), "r"(id) : "memory");
        else if constexpr (KIND == 1)
            asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;" :: "r"(d), "l"(a), "l"(b), "r"(id) : "memory");
        else
            asm volatile("tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, 1;" :: "r"(d), "l"(a), "l"(b), "r"(id) : "memory");
    } else {
        if constexpr (KIND == 0)
            asm volatile("tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, 1;" :: "r"(d), "l"(a), "l"(b), "r"(id) : "memory");
        else if constexpr (KIND == 1)
            asm volatile("tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, 1;" :: "r"(d), "l"(a), "l"(b), "r"(id) : "memory");
        else
            asm volatile("tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], %1, %2, %3, 1;" :: "r"(d), "l"(a), "l"(b), "r"(id) : "memory");
    }
}

// 120 KB of dynamic shared memory keeps it to one CTA per SM (the operands use 48 KB)
constexpr int SMEM = 120 * 1024;

template <int KIND, int CG>
__global__ void __launch_bounds__(128, 1) mma_peak_kernel(int iters) {
    extern __shared__ uint8_t smd[];
    uint8_t *a = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smd) + 1023) & ~uintptr_t(1023));
    uint8_t *b = a + 16384;
    __shared__ uint32_t taddr;
    __shared__ uint64_t bar;
    const int warp = threadIdx.x >> 5;
    // random operand bits (a hash of the position): zero operands draw far
    // less power and would overstate the sustained (power-capped) peak
    for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x) {
        uint32_t x = (uint32_t)i * 2654435761u + blockIdx.x * 40503u;
        x ^= x >> 15; x *= 2246822519u; x ^= x >> 13;
        if (KIND != 0) x &= 0x3F3F3F3Fu;      // bf16 / e4m3: keep exponents moderate (no inf/NaN)
        reinterpret_cast<uint32_t *>(a)[i] = x;
    }
    ptx::fence_async_smem();
    if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_barrier_init(); }
    if (warp == 0) {
        if constexpr (CG == 1) ptx::tmem_alloc<512>(&taddr);
        else ptx::tmem_alloc_pair<512>(&taddr);
    }
    ptx::tc_fence_before();
    if constexpr (CG == 2) ptx::cluster_sync(); else __syncthreads();
    ptx::tc_fence_after();
    const uint32_t rank = CG == 2 ? ptx::cluster_ctarank() : 0;
    if (warp == 0 && rank == 0) {
        constexpr uint32_t ID = idesc<KIND>(128 * CG, 256);
        const uint64_t ad = ptx::sdesc_sw128(ptx::smem_u32(a)), bd = ptx::sdesc_sw128(ptx::smem_u32(b));
        const uint32_t t = taddr;
        for (int it = 0; it < iters; it += 8) {
            if (ptx::elect_one()) {
#pragma unroll
                for (int x = 0; x < 8; x++) mma<KIND, CG>(t + (x & 1) * 256, ad + 2 * ((x >> 1) & 3), bd + 2 * ((x >> 1) & 3), ID);
            }
            __syncwarp();
        }
        if (ptx::elect_one()) {
            if constexpr (CG == 1) ptx::mma_commit(&bar);
            else ptx::mma_commit_pair(&bar, 0x3);
        }
        __syncwarp();
    }
    if (warp == 0 && (CG == 2 || rank == 0)) ptx::mbar_wait(&bar, 0);
    ptx::tc_fence_before();
    if constexpr (CG == 2) ptx::cluster_sync(); else __syncthreads();
    if (warp == 0) {
        if constexpr (CG == 1) ptx::tmem_dealloc<512>(taddr);
        else ptx::tmem_dealloc_pair<512>(taddr);
    }
}

template <int KIND, int CG>
int launch(int ctas, int iters, cudaStream_t st) {
    auto k = mma_peak_kernel<KIND, CG>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)ctas);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CG;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return (int)cudaLaunchKernelEx(&cfg, k, iters);
}

}  // namespace

// One launch on `stream` over `ctas` CTAs (a multiple of cg).  Returns a
// cudaError_t.  K per instruction is 32 bytes (i8 / e4m3: K = 32, bf16: K = 16).
extern "C" int tb_mma_peak_launch(int kind, int cg, int ctas, int iters, void *stream) {
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (cg == 1) {
        if (kind == 0) return launch<0, 1>(ctas, iters, st);
        if (kind == 1) return launch<1, 1>(ctas, iters, st);
        return launch<2, 1>(ctas, iters, st);
    }
    if (kind == 0) return launch<0, 2>(ctas, iters, st);
    if (kind == 1) return launch<1, 2>(ctas, iters, st);
    return launch<2, 2>(ctas, iters, st);
}

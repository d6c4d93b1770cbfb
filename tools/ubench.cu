// Microbenchmarks that bound the tcgen05 kernels (B200, sm_100a):
//   1. tcgen05.ld throughput per SM (32x32b.x16/.x32/.x64; 4/8/16 warps)
//   2. tcgen05.ld throughput while the tensor pipe runs MMAs
//   3. tcgen05.mma issue rates for the shapes sla_tc / w8a8 use
//   4. MUFU ex2 throughput per SM
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/ubench tools/ubench.cu -lcuda
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "../paper_2512_16093_b200/csrc/ptx.cuh"
using namespace tb;

__device__ __forceinline__ void ld32(uint32_t t, uint32_t (&r)[32]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                 "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                   "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
                   "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
                   "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                 : "r"(t));
}

// mode 0: x16 x4, mode 1: x32 x2 per 64 columns
template <int MODE>
__global__ void __launch_bounds__(512, 1) k_ld(int iters, int nwarps, int mma_bg, unsigned long long *out,
                                               unsigned *sink) {
    __shared__ __align__(1024) uint8_t sm[2][16384];
    __shared__ uint32_t taddr;
    __shared__ uint64_t bar;
    __shared__ volatile int stop;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) ptx::tmem_alloc<512>(&taddr);
    if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_barrier_init(); stop = 0; }
    ptx::tc_fence_before(); __syncthreads(); ptx::tc_fence_after();
    uint32_t acc = 0;
    unsigned long long t0 = clock64();
    if (warp < nwarps) {
        const uint32_t base = taddr + ((uint32_t)((warp & 3) * 32) << 16) + ((warp >> 2) & 3) * 64;
        for (int it = 0; it < iters; it++) {
            if (MODE == 0) {
                uint32_t r[4][16];
#pragma unroll
                for (int q = 0; q < 4; q++) ptx::tmem_ld16(base + q * 16, r[q]);
                ptx::tmem_wait_ld();
#pragma unroll
                for (int q = 0; q < 4; q++) acc += r[q][0] ^ r[q][15];
            } else {
                uint32_t r[2][32];
                ld32(base, r[0]);
                ld32(base + 32, r[1]);
                ptx::tmem_wait_ld();
                acc += r[0][0] ^ r[1][31];
            }
        }
    } else if (mma_bg && warp == 15 && (threadIdx.x & 31) == 0) {
        // background MMAs into columns 256..383 (bf16 M128 N128 K16 from smem)
        const uint64_t ad = ptx::sdesc_sw128(ptx::smem_u32(sm[0])), bd = ptx::sdesc_sw128(ptx::smem_u32(sm[1]));
        for (int it = 0; it < iters / 4; it++) {
            for (int k = 0; k < 4; k++) ptx::mma_f16(taddr + 256, ad, bd, ptx::idesc_bf16(128, 128), 1);
            ptx::mma_commit(&bar);
            ptx::mbar_wait(&bar, it & 1);
        }
    }
    __syncthreads();
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    if (acc == 0x12345) sink[0] = acc;
    ptx::tc_fence_before(); __syncthreads();
    if (warp == 0) ptx::tmem_dealloc<512>(taddr);
}

// MMA rate: `iters` groups of 4 K-steps per chain.  KIND 0 = i8 ss, 1 = bf16 ss,
// 2 = bf16 ts (A in TMEM).  WARP=1: the whole warp runs the loop (uniform
// values) and one elected lane issues; WARP=0: lane 0 alone runs it.
template <int KIND, int N, int CHAINS, int RR, int WARP>
__global__ void __launch_bounds__(128, 1) k_mma(int iters, unsigned long long *out) {
    extern __shared__ uint8_t smd[];
    uint8_t (*sm)[32768] = reinterpret_cast<uint8_t (*)[32768]>((reinterpret_cast<uintptr_t>(smd) + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t taddr;
    __shared__ uint64_t bar;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) ptx::tmem_alloc<512>(&taddr);
    if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_barrier_init(); }
    ptx::tc_fence_before(); __syncthreads(); ptx::tc_fence_after();
    unsigned long long t0 = clock64();
    const bool run = WARP ? (warp == 0) : (threadIdx.x == 0);
    if (run) {
        const uint64_t ad = ptx::sdesc_sw128(ptx::smem_u32(sm[0])), bd = ptx::sdesc_sw128(ptx::smem_u32(sm[1]));
        constexpr uint32_t ID = KIND == 0 ? ptx::idesc_i8(128, N) : ptx::idesc_bf16(128, N);
        const uint32_t tb = taddr;
        for (int it = 0; it < iters; it += CHAINS) {
#pragma unroll
            for (int x = 0; x < 4 * CHAINS; x++) {
                const int c = RR ? x % CHAINS : x / 4, k = RR ? x / CHAINS : x % 4;
                const uint32_t dt = tb + c * N;
                if (!WARP || ptx::elect_one()) {
                    if (KIND == 0) ptx::mma_i8(dt, ad + 2 * k, bd + 2 * k, ID, 1);
                    else if (KIND == 1) ptx::mma_f16(dt, ad + 2 * k, bd + 2 * k, ID, 1);
                    else ptx::mma_f16_ts(dt, tb + 448 + 8 * k, bd + 2 * k, ID, 1);
                }
                if (WARP) __syncwarp();
            }
        }
        if (!WARP || ptx::elect_one()) ptx::mma_commit(&bar);
        ptx::mbar_wait(&bar, 0);
    }
    __syncthreads();
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    ptx::tc_fence_before(); __syncthreads();
    if (warp == 0) ptx::tmem_dealloc<512>(taddr);
}

template <int KIND, int N, int CHAINS, int RR, int WARP>
void run_mma(unsigned long long *d) {
    auto f = k_mma<KIND, N, CHAINS, RR, WARP>;
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
    unsigned long long h = 0;
    for (int rep = 0; rep < 2; rep++) { f<<<148, 128, 66 * 1024>>>(1000, d); cudaDeviceSynchronize(); }
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    const char *kn[3] = {"i8 ss", "bf16 ss", "bf16 ts"};
    const double macs = 1000.0 * 4 * 128 * N * (KIND == 0 ? 32 : 16);
    printf("mma %-7s M128 N%3d chains %d %-11s %s: %6.1f clk/mma, %5.0f MAC/clk/SM\n", kn[KIND], N, CHAINS,
           RR ? "interleaved" : "sequential", WARP ? "warp+elect" : "lane0     ", (double)h / 4000, macs / h);
}

__global__ void __launch_bounds__(1024, 1) k_mufu(int iters, unsigned long long *out, float *sink) {
    float x0 = threadIdx.x * 1e-3f, x1 = x0 + 0.1f, x2 = x0 + 0.2f, x3 = x0 + 0.3f;
    __syncthreads();
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x0));
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x1));
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x2));
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x3));
    }
    __syncthreads();
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    if (x0 + x1 + x2 + x3 == 1.2345f) sink[0] = x0;
}

// ex2 variants: f32, f16x2, bf16x2 (4 independent chains per thread)
template <int V>
__global__ void __launch_bounds__(1024, 1) k_ex2(int iters, unsigned long long *out, unsigned *sink) {
    uint32_t x0 = threadIdx.x * 7u, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
    __syncthreads();
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
        if (V == 0) {
            asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+r"(x0)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+r"(x1));
            asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+r"(x2)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+r"(x3));
        } else if (V == 1) {
            asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(x0)); asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(x1));
            asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(x2)); asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(x3));
        } else if (V == 2) {
            asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(x0)); asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(x1));
            asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(x2)); asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(x3));
        } else if (V == 3) {   // f32 pair -> f16x2 convert (F2FP)
            asm volatile("cvt.rn.f16x2.f32 %0, %0, %1;" : "+r"(x0) : "r"(x1)); asm volatile("cvt.rn.f16x2.f32 %0, %0, %1;" : "+r"(x1) : "r"(x2));
            asm volatile("cvt.rn.f16x2.f32 %0, %0, %1;" : "+r"(x2) : "r"(x3)); asm volatile("cvt.rn.f16x2.f32 %0, %0, %1;" : "+r"(x3) : "r"(x0));
        } else {               // HADD2
            asm volatile("add.rn.f16x2 %0, %0, %1;" : "+r"(x0) : "r"(x1)); asm volatile("add.rn.f16x2 %0, %0, %1;" : "+r"(x1) : "r"(x2));
            asm volatile("add.rn.f16x2 %0, %0, %1;" : "+r"(x2) : "r"(x3)); asm volatile("add.rn.f16x2 %0, %0, %1;" : "+r"(x3) : "r"(x0));
        }
    }
    __syncthreads();
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    if ((x0 ^ x1 ^ x2 ^ x3) == 0x12345) sink[0] = x0;
}
template <int V>
void run_ex2(unsigned long long *d, unsigned *s, const char *name) {
    unsigned long long h = 0;
    for (int rep = 0; rep < 2; rep++) { k_ex2<V><<<148, 1024>>>(1000, d, s); cudaDeviceSynchronize(); }
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("%-22s: %.2f warp-instr per clk per SM (%.1f thread-ops/clk/SM)\n", name, 1000.0 * 4 * 32 / h, 1000.0 * 4 * 1024 / h);
}

int main() {
    unsigned long long *d, h;
    unsigned *s;
    float *sf;
    cudaMalloc(&d, 8 * 148);
    cudaMalloc(&s, 4);
    cudaMalloc(&sf, 4);
    const int iters = 4000;
    run_ex2<0>(d, s, "ex2.approx.ftz.f32");
    run_ex2<1>(d, s, "ex2.approx.f16x2");
    run_ex2<2>(d, s, "ex2.approx.ftz.bf16x2");
    run_ex2<3>(d, s, "cvt.rn.f16x2.f32");
    run_ex2<4>(d, s, "add.rn.f16x2");
    if (getenv("SKIP_MMA") != nullptr) return 0;
    if (getenv("SKIP_LD") == nullptr)
    for (int bg : {0, 1})
        for (int mode : {0, 1})
            for (int nw : {1, 4, 8, 12, 16}) {
                if (bg && nw == 16) continue;
                for (int rep = 0; rep < 2; rep++) {
                    if (mode == 0) k_ld<0><<<148, 512>>>(iters, nw, bg, d, s);
                    else k_ld<1><<<148, 512>>>(iters, nw, bg, d, s);
                    cudaDeviceSynchronize();
                }
                cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
                const double bytes = (double)iters * nw * 32 * 64 * 4;
                printf("tmem_ld %s warps %2d mma_bg %d: %.1f B/clk/SM  (%.1f clk per 64-col 8KB warp load)\n",
                       mode ? "x32" : "x16", nw, bg, bytes / h, (double)h * nw / iters / nw);
            }
    run_mma<0, 64, 1, 0, 0>(d);
    run_mma<0, 64, 1, 0, 1>(d);
    run_mma<0, 64, 2, 0, 0>(d);
    run_mma<0, 64, 2, 0, 1>(d);
    run_mma<0, 64, 2, 1, 0>(d);
    run_mma<0, 64, 2, 1, 1>(d);
    run_mma<0, 128, 1, 0, 0>(d);
    run_mma<0, 128, 1, 0, 1>(d);
    run_mma<0, 128, 2, 0, 0>(d);
    run_mma<0, 128, 2, 0, 1>(d);
    run_mma<0, 128, 2, 1, 0>(d);
    run_mma<0, 128, 2, 1, 1>(d);
    run_mma<0, 256, 1, 0, 0>(d);
    run_mma<0, 256, 1, 0, 1>(d);
    run_mma<0, 256, 2, 0, 0>(d);
    run_mma<0, 256, 2, 0, 1>(d);
    run_mma<0, 256, 2, 1, 0>(d);
    run_mma<0, 256, 2, 1, 1>(d);
    run_mma<2, 64, 1, 0, 0>(d);
    run_mma<2, 64, 1, 0, 1>(d);
    run_mma<2, 64, 2, 0, 0>(d);
    run_mma<2, 64, 2, 0, 1>(d);
    run_mma<2, 64, 2, 1, 0>(d);
    run_mma<2, 64, 2, 1, 1>(d);
    run_mma<2, 128, 1, 0, 0>(d);
    run_mma<2, 128, 1, 0, 1>(d);
    run_mma<2, 128, 2, 0, 0>(d);
    run_mma<2, 128, 2, 0, 1>(d);
    run_mma<2, 128, 2, 1, 0>(d);
    run_mma<2, 128, 2, 1, 1>(d);
    run_mma<2, 256, 1, 0, 0>(d);
    run_mma<2, 256, 1, 0, 1>(d);
    run_mma<1, 256, 1, 0, 1>(d);
    for (int rep = 0; rep < 2; rep++) { k_mufu<<<148, 1024>>>(1000, d, sf); cudaDeviceSynchronize(); }
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("mufu ex2: %.2f per clk per SM\n", 1000.0 * 4 * 1024 / h);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}

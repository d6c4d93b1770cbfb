// Per-SMSP issue rates of the softmax instruction mix (B200, sm_100a).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_alu tools/ubench_alu.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

template <int OP>
__global__ void __launch_bounds__(1024, 1) k(int iters, unsigned long long *out, uint32_t *sink) {
    uint32_t r[8];
    for (int i = 0; i < 8; i++) r[i] = threadIdx.x * 13 + i;
    unsigned long long c = 0x3f8000003f800000ull;
    __syncthreads();
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) {
            if (OP == 0) asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+r"(r[i]));
            if (OP == 1) {  // FFMA2 on a register pair
                unsigned long long v = ((unsigned long long)r[i] << 32) | r[(i + 1) & 7];
                asm volatile("fma.rn.f32x2 %0, %0, %1, %0;" : "+l"(v) : "l"(c));
                r[i] = (uint32_t)v;
            }
            if (OP == 2) asm volatile("add.u32 %0, %0, 0x4b400000;" : "+r"(r[i]));
            if (OP == 3) asm volatile("max.f32 %0, %0, %1;" : "+r"(r[i]) : "r"(r[(i + 3) & 7]));
            if (OP == 4) asm volatile("{.reg .b32 t; cvt.rn.bf16x2.f32 t, %0, %1; mov.b32 %0, t;}" : "+r"(r[i]) : "r"(r[(i + 1) & 7]));
            if (OP == 5) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+r"(r[i]));
            if (OP == 6) asm volatile("mad.lo.u32 %0, %0, 0x800000, %1;" : "+r"(r[i]) : "r"(r[(i + 1) & 7]));
            if (OP == 8) asm volatile("cvt.rn.f32.s32 %0, %0;" : "+r"(r[i]));
            if (OP == 9) {  // FADD2 on a register pair
                unsigned long long v = ((unsigned long long)r[i] << 32) | r[(i + 1) & 7];
                asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(v) : "l"(c));
                r[i] = (uint32_t)v;
            }
            if (OP == 10) {  // W8A8 epilogue pair: 2 x I2F + FFMA2
                asm volatile("cvt.rn.f32.s32 %0, %0;" : "+r"(r[i]));
                asm volatile("cvt.rn.f32.s32 %0, %0;" : "+r"(r[(i + 1) & 7]));
                unsigned long long v = ((unsigned long long)r[(i + 2) & 7] << 32) | r[(i + 3) & 7];
                asm volatile("fma.rn.f32x2 %0, %0, %1, %0;" : "+l"(v) : "l"(c));
                r[(i + 2) & 7] = (uint32_t)v;
            }
            if (OP == 7) {  // mix: 1 ex2 + 2 ffma2 + 1 add + 1 f2fp per "element pair"
                unsigned long long v = ((unsigned long long)r[i] << 32) | r[(i + 1) & 7];
                asm volatile("fma.rn.f32x2 %0, %0, %1, %0;" : "+l"(v) : "l"(c));
                asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(v) : "l"(c));
                r[i] = (uint32_t)v;
                asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+r"(r[i]));
                asm volatile("add.u32 %0, %0, 0x4b400000;" : "+r"(r[(i + 2) & 7]));
                asm volatile("{.reg .b32 t; cvt.rn.bf16x2.f32 t, %0, %1; mov.b32 %0, t;}" : "+r"(r[(i + 4) & 7]) : "r"(r[(i + 5) & 7]));
            }
        }
    }
    __syncthreads();
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    uint32_t x = 0;
    for (int i = 0; i < 8; i++) x ^= r[i];
    if (x == 0x12345) sink[0] = x;
}

template <int OP>
void run(const char *name, int nthreads, double instr_per_iter) {
    unsigned long long *d, h;
    uint32_t *s;
    cudaMalloc(&d, 8 * 148);
    cudaMalloc(&s, 4);
    for (int rep = 0; rep < 2; rep++) { k<OP><<<148, nthreads>>>(1000, d, s); cudaDeviceSynchronize(); }
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    const double warps_per_smsp = nthreads / 32 / 4.0;
    printf("%-28s threads %4d: %.3f warp-instr/clk/SMSP\n", name, nthreads, 1000.0 * instr_per_iter * warps_per_smsp / h);
    cudaFree(d);
    cudaFree(s);
}

int main() {
    for (int nt : {256, 1024}) {
        run<0>("FFMA", nt, 8);
        run<1>("FFMA2", nt, 8);
        run<2>("IADD (magic)", nt, 8);
        run<3>("FMNMX", nt, 8);
        run<4>("F2FP.BF16.PACK", nt, 8);
        run<5>("MUFU.EX2", nt, 8);
        run<6>("IMAD", nt, 8);
        run<7>("mix (ffma2,fadd2,ex2,iadd,f2fp)", nt, 40);
        run<8>("I2F (cvt.rn.f32.s32)", nt, 8);
        run<9>("FADD2", nt, 8);
        run<10>("2 I2F + FFMA2", nt, 24);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}

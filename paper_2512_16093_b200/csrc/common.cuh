// common.cuh -- shared device helpers for the sm_100a hot-path kernels.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <string>

#include "../../include/tb_capi.h"

namespace tb {

// ---------------------------------------------------------------- errors
void set_error(const std::string &msg);
int fail(int code, const std::string &msg);
int check_launch(const char *what);

#define TB_REQUIRE(cond, msg) \
    do { if (!(cond)) return ::tb::fail(TB_EINVAL, (msg)); } while (0)

int ensure_smem(const void *fn, int bytes);
template <typename F>
inline void smem_attr(F *kern, int bytes) { ensure_smem(reinterpret_cast<const void *>(kern), bytes); }

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// ----------------------------------------------------------- load helpers
template <typename T> __device__ __forceinline__ float to_f32(T v);
template <> __device__ __forceinline__ float to_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 v) {
    return __bfloat162float(v);
}

// The reference quantization rule (attention.py:215-219, blockquant.py:106-109):
// scale = f32(f64(am)/127) == __fdiv_rn(am, 127) (double rounding innocuous for
// division at 53 >= 2*24+2 bits); code = clip(rint(x/safe), -127, 127), IEEE divide.
__device__ __forceinline__ float quant_scale(float am) { return __fdiv_rn(am, 127.0f); }
__device__ __forceinline__ int8_t quant_code(float x, float safe) {
    float r = rintf(__fdiv_rn(x, safe));
    r = fminf(fmaxf(r, -127.0f), 127.0f);
    return (int8_t)(int)r;
}

// Same code as quant_code for |x| <= 127 * safe, from one FMA against inv =
// __frcp_rn(safe): u = M + rint(x * inv) (M = 1.5*2^23); x * inv is within
// 1.2e-5 of the IEEE quotient fl(x / safe), so unless x * inv lands within
// 2^-15 of a rounding boundary (probability ~6e-5) both round to the same
// integer; near a boundary the exact division decides.  Returns the int8
// code in the low byte.
__device__ __forceinline__ uint32_t quant_code_fast(float x, float safe, float inv) {
    const float u = __fmaf_rn(x, inv, 12582912.0f);
    const float w = __fsub_rn(u, 12582912.0f);
    const float dlt = __fmaf_rn(x, inv, -w);
    if (fabsf(dlt) > 0.5f - 0x1p-15f) return (uint32_t)(uint8_t)quant_code(x, safe);
    return (uint32_t)__float_as_int(u) & 0xFFu;
}

// quant_code_fast for N (multiple of 4) values packed into N/4 words
// (little-endian bytes), branch-free on the common path: the rare near-tie
// elements (|dlt| within 2^-15 of 0.5) are collected in a mask and redone with
// the exact division afterwards, so the unrolled loop carries no per-element
// branch.
template <int N>
__device__ __forceinline__ void quant_fast_n(const float (&x)[N], float safe, float inv, bool exact_all,
                                             uint32_t (&w)[N / 4]) {
    uint32_t need = 0u;
#pragma unroll
    for (int k = 0; k < N / 4; k++) w[k] = 0u;
#pragma unroll
    for (int i = 0; i < N; i++) {
        const float u = __fmaf_rn(x[i], inv, 12582912.0f);
        const float t = __fsub_rn(u, 12582912.0f);
        const float dlt = __fmaf_rn(x[i], inv, -t);
        need |= (uint32_t)(fabsf(dlt) > 0.5f - 0x1p-15f) << i;
        w[i >> 2] |= ((uint32_t)__float_as_int(u) & 0xFFu) << ((i & 3) * 8);
    }
    if (exact_all) need = ~0u;
    if (need) {
#pragma unroll
        for (int i = 0; i < N; i++) {             // static indices keep x[] in registers
            if ((need >> i) & 1u) {
                const uint32_t c8 = (uint32_t)(uint8_t)quant_code(x[i], safe);
                const int sh = (i & 3) * 8;
                w[i >> 2] = (w[i >> 2] & ~(0xFFu << sh)) | (c8 << sh);
            }
        }
    }
}
__device__ __forceinline__ void quant16_fast(const float (&x)[16], float safe, float inv, bool exact_all,
                                             uint32_t (&w)[4]) {
    quant_fast_n<16>(x, safe, inv, exact_all, w);
}

template <int N>
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Block-wide max of non-negative floats (absmax); `red` needs 32 floats.
__device__ __forceinline__ float block_max_nonneg(float v, float *red) {
    v = warp_max<32>(v);
    int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    int nw = (blockDim.x + 31) >> 5;
    float r = (l < nw) ? red[l] : 0.0f;
    r = warp_max<32>(r);
    return r;
}

__host__ __device__ inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace tb

namespace tb {
__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
}  // namespace tb

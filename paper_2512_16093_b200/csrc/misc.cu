// misc.cu -- elementwise / row kernels around the hot path:
//   feature map phi (attention.py:287-290) into padded GEMM operands,
//   rmsnorm / layernorm / gelu (sampler.py:34-58) for the DiT block,
//   error/info plumbing of the C ABI.
#include <cstdio>
#include <string>

#include "common.cuh"

namespace tb {

static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }
int fail(int code, const std::string &msg) {
    set_error(msg);
    return code;
}
int check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(TB_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
    return TB_OK;
}

__device__ __forceinline__ float phi(float x) { return x >= 0.0f ? x + 1.0f : expf(x); }

// phi(x) [H,L,d] -> out [H,l_pad,d] (bf16 or f32), rows >= L zero (padding
// rows must contribute nothing to phi(K)^T V, and phi(0) = 1 != 0).
template <typename T, typename O>
__global__ void feature_map_kernel(const T *__restrict__ x, int64_t H, int64_t L, int64_t d, int64_t l_pad,
                                   O *__restrict__ out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t n = H * l_pad * d;
    if (i >= n) return;
    int64_t c = i % d, t = (i / d) % l_pad, h = i / (d * l_pad);
    float r = (t < L) ? phi(to_f32(x[(h * L + t) * d + c])) : 0.0f;
    if constexpr (sizeof(O) == 2) out[i] = __float2bfloat16_rn(r);
    else out[i] = r;
}

// one warp per row
__global__ void rmsnorm_kernel(const float *__restrict__ x, const float *__restrict__ g, int64_t rows,
                               int64_t cols, float eps, float *__restrict__ out) {
    int64_t row = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
    int lane = threadIdx.x & 31;
    if (row >= rows) return;
    const float *xr = x + row * cols;
    float s = 0.0f;
    for (int64_t c = lane; c < cols; c += 32) s = fmaf(xr[c], xr[c], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const float inv = 1.0f / sqrtf(s / (float)cols + eps);
    for (int64_t c = lane; c < cols; c += 32) out[row * cols + c] = xr[c] * inv * g[c];
}

__global__ void layernorm_kernel(const float *__restrict__ x, const float *__restrict__ g,
                                 const float *__restrict__ b, int64_t rows, int64_t cols, float eps,
                                 float *__restrict__ out) {
    int64_t row = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
    int lane = threadIdx.x & 31;
    if (row >= rows) return;
    const float *xr = x + row * cols;
    float s = 0.0f;
    for (int64_t c = lane; c < cols; c += 32) s += xr[c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const float mu = s / (float)cols;
    float v = 0.0f;
    for (int64_t c = lane; c < cols; c += 32) { float t = xr[c] - mu; v = fmaf(t, t, v); }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const float inv = 1.0f / sqrtf(v / (float)cols + eps);
    for (int64_t c = lane; c < cols; c += 32) out[row * cols + c] = (xr[c] - mu) * inv * g[c] + b[c];
}

__global__ void gelu_kernel(const float *__restrict__ x, int64_t n, float *__restrict__ out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float c = 0.7978845608028654f;  // sqrt(2/pi)
    float v = x[i];
    out[i] = 0.5f * v * (1.0f + tanhf(c * (v + 0.044715f * v * v * v)));
}

}  // namespace tb

using namespace tb;

extern "C" const char *tb_last_error(void) { return g_last_error.c_str(); }

extern "C" const char *tb_build_info(void) {
    return "tb200: sm_100a (tcgen05 kind::i8 / kind::f16, TMA tensor + bulk copies)";
}

extern "C" int tb_device_ok(void) {
    int dev = 0, major = 0, minor = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    return (major == 10 && minor == 0) ? 1 : 0;
}

extern "C" int tb_feature_map(const void *x, int dtype, int64_t H, int64_t L, int64_t d, int64_t l_pad,
                              void *out, int out_dtype, void *stream) {
    TB_REQUIRE(l_pad >= L, "l_pad < L");
    int64_t n = H * l_pad * d;
    if (n == 0) return TB_OK;
    unsigned grid = (unsigned)cdiv(n, 256);
    cudaStream_t st = as_stream(stream);
    if (dtype == TB_F32 && out_dtype == TB_BF16)
        feature_map_kernel<float, __nv_bfloat16><<<grid, 256, 0, st>>>((const float *)x, H, L, d, l_pad, (__nv_bfloat16 *)out);
    else if (dtype == TB_F32)
        feature_map_kernel<float, float><<<grid, 256, 0, st>>>((const float *)x, H, L, d, l_pad, (float *)out);
    else if (out_dtype == TB_BF16)
        feature_map_kernel<__nv_bfloat16, __nv_bfloat16><<<grid, 256, 0, st>>>((const __nv_bfloat16 *)x, H, L, d, l_pad, (__nv_bfloat16 *)out);
    else
        feature_map_kernel<__nv_bfloat16, float><<<grid, 256, 0, st>>>((const __nv_bfloat16 *)x, H, L, d, l_pad, (float *)out);
    return check_launch("feature_map");
}

extern "C" int tb_rmsnorm(const float *x, const float *gain, int64_t rows, int64_t cols, float eps, float *out,
                          void *stream) {
    TB_REQUIRE(eps > 0.0f, "eps must be > 0");
    if (rows == 0) return TB_OK;
    rmsnorm_kernel<<<(unsigned)cdiv(rows, 8), 256, 0, as_stream(stream)>>>(x, gain, rows, cols, eps, out);
    return check_launch("rmsnorm");
}

extern "C" int tb_layernorm(const float *x, const float *gain, const float *offset, int64_t rows, int64_t cols,
                            float eps, float *out, void *stream) {
    TB_REQUIRE(eps > 0.0f, "eps must be > 0");
    if (rows == 0) return TB_OK;
    layernorm_kernel<<<(unsigned)cdiv(rows, 8), 256, 0, as_stream(stream)>>>(x, gain, offset, rows, cols, eps, out);
    return check_launch("layernorm");
}

extern "C" int tb_gelu(const float *x, int64_t n, float *out, void *stream) {
    if (n == 0) return TB_OK;
    gelu_kernel<<<(unsigned)cdiv(n, 256), 256, 0, as_stream(stream)>>>(x, n, out);
    return check_launch("gelu");
}

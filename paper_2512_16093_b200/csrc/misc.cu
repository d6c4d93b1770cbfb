// misc.cu -- elementwise / row kernels around the hot path:
//   feature map phi (attention.py:287-290) into padded GEMM operands,
//   rmsnorm / layernorm / gelu (sampler.py:34-58) for the DiT block,
//   error/info plumbing of the C ABI.
#include <cstdio>
#include <mutex>
#include <map>
#include <string>
#include <utility>

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

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) only when a launch needs
// more than the kernel's current limit: the attribute is a sticky per-device
// maximum, so once raised it covers every smaller launch and the launch path
// pays a locked map lookup instead of a driver call.
int ensure_smem(const void *fn, int bytes) {
    static std::mutex mu;
    static std::map<std::pair<int, const void *>, int> limit;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(mu);
    int &cur = limit[std::make_pair(dev, fn)];
    if (bytes <= cur) return 0;
    const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) cur = bytes;
    return (int)e;
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

// One pass over q, k, v producing every operand the SLA pipeline derives
// from the raw tensors besides codes/pools (attention.py:306-334 and the PV
// B operand), in the GEMM dtype O (bf16 or f32):
//   phiq [H,lq,d]  phi(q), zero rows t >= L                  (may be NULL)
//   phik [H,lk,d]  phi(k), zero rows t >= L: padding rows must contribute
//                  nothing to phi(K)^T V (phi(0) = 1 != 0)     (may be NULL)
//   vext [H,lk,dx] [v | 1 | 0...]: the ones column makes phi(K)^T vext carry
//                  sum_t phi(k_t), the denominator term, in column d
//   vt   [H,d,lvt] bf16 V^T, zero padded (K-major B operand of the PV MMA)
// CTA = one head x 64 tokens; thread = 8 channels of one token row; V^T is
// transposed through shared memory (row pitch d+2 keeps it conflict-free).
template <typename T, typename O>
__global__ void __launch_bounds__(256) linear_operands_kernel(
    const T *__restrict__ q, const T *__restrict__ k, const T *__restrict__ v, int64_t L, int d, int64_t lq,
    int64_t lk, int dx, O *__restrict__ phiq, O *__restrict__ phik, O *__restrict__ vext,
    __nv_bfloat16 *__restrict__ vt, int64_t lvt) {
    extern __shared__ __align__(16) __nv_bfloat16 vs[];   // [64][d+2]
    const int64_t h = blockIdx.y;
    const int64_t t0 = blockIdx.x * 64LL;
    const int cg = d / 8;
    const int rows = blockDim.x / cg;
    const int tx = threadIdx.x % cg, ty = threadIdx.x / cg;
    const int c0 = tx * 8;
    auto st = [](O *dst, const float *x) {
        if constexpr (sizeof(O) == 2) {
            uint4 w;
            __nv_bfloat162 *p = reinterpret_cast<__nv_bfloat162 *>(&w);
#pragma unroll
            for (int i = 0; i < 4; i++) p[i] = __floats2bfloat162_rn(x[2 * i], x[2 * i + 1]);
            *reinterpret_cast<uint4 *>(dst) = w;
        } else {
            *reinterpret_cast<float4 *>(dst) = make_float4(x[0], x[1], x[2], x[3]);
            *reinterpret_cast<float4 *>(dst + 4) = make_float4(x[4], x[5], x[6], x[7]);
        }
    };
    auto ld = [&](const T *src, float *x, bool in) {
        if (!in) {
#pragma unroll
            for (int i = 0; i < 8; i++) x[i] = 0.0f;
            return;
        }
        if constexpr (sizeof(T) == 2) {
            uint4 w = *reinterpret_cast<const uint4 *>(src);
            const __nv_bfloat162 *p = reinterpret_cast<const __nv_bfloat162 *>(&w);
#pragma unroll
            for (int i = 0; i < 4; i++) { float2 f = __bfloat1622float2(p[i]); x[2 * i] = f.x; x[2 * i + 1] = f.y; }
        } else {
            float4 a = *reinterpret_cast<const float4 *>(src), b = *reinterpret_cast<const float4 *>(src + 4);
            x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w; x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
        }
    };
    const int pitch = d + 2;
    for (int tr = ty; tr < 64; tr += rows) {
        const int64_t t = t0 + tr;
        const bool in = t < L;
        const int64_t off = (h * L + (in ? t : 0)) * d + c0;
        float xv[8];
        ld(v + off, xv, in);
        if (vt) {
#pragma unroll
            for (int i = 0; i < 8; i++) vs[tr * pitch + c0 + i] = __float2bfloat16_rn(xv[i]);
        }
        if (phiq && t < lq) {
            float xq[8];
            ld(q + off, xq, in);
#pragma unroll
            for (int i = 0; i < 8; i++) xq[i] = in ? phi(xq[i]) : 0.0f;
            st(phiq + (h * lq + t) * d + c0, xq);
        }
        if (phik && t < lk) {
            float xk[8];
            ld(k + off, xk, in);
#pragma unroll
            for (int i = 0; i < 8; i++) xk[i] = in ? phi(xk[i]) : 0.0f;
            st(phik + (h * lk + t) * d + c0, xk);
            st(vext + (h * lk + t) * dx + c0, xv);
            if (tx == 0) {
                float e[8] = {in ? 1.0f : 0.0f, 0, 0, 0, 0, 0, 0, 0};
                for (int c = d; c < dx; c += 8) {
                    st(vext + (h * lk + t) * dx + c, e);
                    e[0] = 0.0f;
                }
            }
        }
    }
    if (!vt || t0 >= lvt) return;
    __syncthreads();
    // V^T rows: channel c, 64 tokens = 8 chunks of 8 tokens (16 B each)
    for (int i = threadIdx.x; i < d * 8; i += blockDim.x) {
        const int c = i >> 3, tc = (i & 7) * 8;
        if (t0 + tc >= lvt) continue;
        uint4 w;
        uint16_t *p = reinterpret_cast<uint16_t *>(&w);
#pragma unroll
        for (int j = 0; j < 8; j++) p[j] = __bfloat16_as_ushort(vs[(tc + j) * pitch + c]);
        *reinterpret_cast<uint4 *>(vt + (h * d + c) * lvt + t0 + tc) = w;
    }
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

// DiT glue in one pass (dit.py): s = x (+ y) (+ alpha * emb), optionally
// stored (f32), and its RMSNorm (MODE 0, sampler.py:34-44) or LayerNorm
// (MODE 1, sampler.py:47-53) as bf16 for the next W8A8 projection.  One CTA
// per row, 256 threads, each thread 4-float chunks kept in registers
// (cols <= 256 * 4 * ADD_NORM_CHUNKS).
constexpr int ADD_NORM_CHUNKS = 8;
// five CTAs per SM (48 registers): RMSNorm 1.34 -> 1.17 ms and LayerNorm
// 1.67 -> 1.21 ms for add_norm + the blockwise quantizer at cfg5 (four: 1.22 /
// 1.25; tools/time_add_norm.py, interleaved A/B)
#ifndef TB_ADDNORM_MINB
#define TB_ADDNORM_MINB 5
#endif
template <int MODE>
__global__ void __launch_bounds__(256, TB_ADDNORM_MINB) add_norm_kernel(
    const float *__restrict__ x, const float *__restrict__ y, const float *__restrict__ emb, float alpha,
    const float *__restrict__ g, const float *__restrict__ b, int64_t cols, float eps, float *__restrict__ sum_out,
    __nv_bfloat16 *__restrict__ norm_out) {
    __shared__ float red[2][8];
    const int64_t row = blockIdx.x;
    const int nc4 = (int)(cols >> 2);
    float4 v[ADD_NORM_CHUNKS];
    float s1 = 0.0f, s2 = 0.0f;
#pragma unroll
    for (int i = 0; i < ADD_NORM_CHUNKS; i++) {
        const int c4 = threadIdx.x + i * 256;
        if (c4 < nc4) {
            float4 a = reinterpret_cast<const float4 *>(x + row * cols)[c4];
            if (y) {
                const float4 t = reinterpret_cast<const float4 *>(y + row * cols)[c4];
                a.x += t.x; a.y += t.y; a.z += t.z; a.w += t.w;
            }
            if (emb) {
                const float4 e = reinterpret_cast<const float4 *>(emb)[c4];
                a.x = fmaf(alpha, e.x, a.x); a.y = fmaf(alpha, e.y, a.y);
                a.z = fmaf(alpha, e.z, a.z); a.w = fmaf(alpha, e.w, a.w);
            }
            if (sum_out) reinterpret_cast<float4 *>(sum_out + row * cols)[c4] = a;
            v[i] = a;
            s1 += (a.x + a.y) + (a.z + a.w);
            s2 = fmaf(a.x, a.x, fmaf(a.y, a.y, fmaf(a.z, a.z, fmaf(a.w, a.w, s2))));
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) { red[0][w] = s1; red[1][w] = s2; }
    __syncthreads();
    s1 = 0.0f; s2 = 0.0f;
#pragma unroll
    for (int i = 0; i < 8; i++) { s1 += red[0][i]; s2 += red[1][i]; }
    const float n = (float)cols;
    float mu = 0.0f, inv;
    if (MODE == 0) {
        inv = rsqrtf(s2 / n + eps);
    } else {
        // population variance in a second pass over the registers (no E[x^2] - mu^2 cancellation)
        mu = s1 / n;
        float s3 = 0.0f;
#pragma unroll
        for (int i = 0; i < ADD_NORM_CHUNKS; i++) {
            if (threadIdx.x + i * 256 < nc4) {
                const float dx = v[i].x - mu, dy = v[i].y - mu, dz = v[i].z - mu, dw = v[i].w - mu;
                s3 = fmaf(dx, dx, fmaf(dy, dy, fmaf(dz, dz, fmaf(dw, dw, s3))));
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s3 += __shfl_xor_sync(0xffffffffu, s3, o);
        __syncthreads();
        if ((threadIdx.x & 31) == 0) red[0][w] = s3;
        __syncthreads();
        s3 = 0.0f;
#pragma unroll
        for (int i = 0; i < 8; i++) s3 += red[0][i];
        inv = rsqrtf(s3 / n + eps);
    }
#pragma unroll
    for (int i = 0; i < ADD_NORM_CHUNKS; i++) {
        const int c4 = threadIdx.x + i * 256;
        if (c4 < nc4) {
            const float4 gg = reinterpret_cast<const float4 *>(g)[c4];
            float4 o;
            o.x = (v[i].x - mu) * inv * gg.x; o.y = (v[i].y - mu) * inv * gg.y;
            o.z = (v[i].z - mu) * inv * gg.z; o.w = (v[i].w - mu) * inv * gg.w;
            if (MODE == 1) {
                const float4 bb = reinterpret_cast<const float4 *>(b)[c4];
                o.x += bb.x; o.y += bb.y; o.z += bb.z; o.w += bb.w;
            }
            __nv_bfloat162 p0 = __floats2bfloat162_rn(o.x, o.y), p1 = __floats2bfloat162_rn(o.z, o.w);
            uint2 wv;
            wv.x = *reinterpret_cast<uint32_t *>(&p0);
            wv.y = *reinterpret_cast<uint32_t *>(&p1);
            reinterpret_cast<uint2 *>(norm_out + row * cols)[c4] = wv;
        }
    }
}


// add_norm + quantize_blockwise(., 128) of its bf16 output in ONE pass over
// HBM (the norm-fed activation quantizations of the DiT block,
// RMSNorm -> qkv and LayerNorm -> mlp_in, sampler.py:161,180).  A 128-row
// quantization band is one cluster of 8 CTAs, 16 rows each (one warp per
// row): pass A forms s = x (+ y) (+ alpha*emb) (stored when sum_out) and the
// row statistics, pass B normalises (s re-read from L2) into a bf16 copy of
// the CTA's rows in shared memory and the per-128-column absmax of those 16
// rows, the band's block maxima are combined across the cluster through
// distributed shared memory, and pass C writes the int8 codes from shared
// memory.  HBM: x, y read once, s and the codes written once (13 B per
// element instead of the two-kernel 17 B: no bf16 round trip).
// The row reduction reproduces add_norm_kernel exactly (virtual thread t =
// lane + 32k holds chunks t + 256 i; per-virtual-warp xor shuffles; the 8
// partials summed in order), so the bf16 values -- and therefore the codes
// and scales -- are bit-identical to tb_add_norm followed by
// tb_quantize_blockwise.
constexpr int ANQ_ROWS = 16, ANQ_CLUSTER = 8;
template <int MODE>
__global__ void __cluster_dims__(ANQ_CLUSTER, 1, 1) __launch_bounds__(ANQ_ROWS * 32, 1) add_norm_quant_kernel(
    const float *__restrict__ x, const float *__restrict__ y, const float *__restrict__ emb, float alpha,
    const float *__restrict__ g, const float *__restrict__ b, int64_t rows, int cols, float eps,
    float *__restrict__ sum_out, int8_t *__restrict__ q, float *__restrict__ scales) {
    extern __shared__ __align__(16) uint8_t anq_smem[];
    const int nc4 = cols >> 2, nb = cols >> 7;
    __nv_bfloat16 *a_s = reinterpret_cast<__nv_bfloat16 *>(anq_smem);                       // [16][cols]
    float *amax = reinterpret_cast<float *>(anq_smem + (size_t)ANQ_ROWS * cols * 2);         // [16][nb]
    float *bmax = amax + ANQ_ROWS * nb;                                                       // [nb] CTA maxima
    float *bsc = bmax + nb;                                                                   // [nb] band scales
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const int64_t band = blockIdx.x / ANQ_CLUSTER;
    const int64_t row = band * 128 + (int64_t)rank * ANQ_ROWS + warp;
    const bool ok = row < rows;
    auto load_s = [&](int c4) {
        float4 a = reinterpret_cast<const float4 *>(x + row * cols)[c4];
        if (y) {
            const float4 t = reinterpret_cast<const float4 *>(y + row * cols)[c4];
            a.x += t.x; a.y += t.y; a.z += t.z; a.w += t.w;
        }
        if (emb) {
            const float4 e = reinterpret_cast<const float4 *>(emb)[c4];
            a.x = fmaf(alpha, e.x, a.x); a.y = fmaf(alpha, e.y, a.y);
            a.z = fmaf(alpha, e.z, a.z); a.w = fmaf(alpha, e.w, a.w);
        }
        return a;
    };
    // s again in pass B: from the stored sum (an L2 hit) or recomputed (same ops)
    auto reload_s = [&](int c4) {
        return sum_out ? reinterpret_cast<const float4 *>(sum_out + row * cols)[c4] : load_s(c4);
    };
    auto xor_sum = [&](float v) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        return v;
    };
    if (ok) {
        // pass A: s, sum_out, row statistics in add_norm_kernel's order
        float s1 = 0.0f, s2 = 0.0f;
#pragma unroll 1
        for (int k = 0; k < 8; k++) {                      // virtual warp k: threads 32k + lane
            float p1 = 0.0f, p2 = 0.0f;
#pragma unroll
            for (int i = 0; i < ADD_NORM_CHUNKS; i++) {
                const int c4 = lane + 32 * k + 256 * i;
                if (c4 < nc4) {
                    const float4 a = load_s(c4);
                    if (sum_out) reinterpret_cast<float4 *>(sum_out + row * cols)[c4] = a;
                    p1 += (a.x + a.y) + (a.z + a.w);
                    p2 = fmaf(a.x, a.x, fmaf(a.y, a.y, fmaf(a.z, a.z, fmaf(a.w, a.w, p2))));
                }
            }
            s1 += xor_sum(p1);                             // 0 + red[0] + red[1] + ... in order
            s2 += xor_sum(p2);
        }
        const float n = (float)cols;
        float mu = 0.0f, inv;
        if (MODE == 0) {
            inv = rsqrtf(s2 / n + eps);
        } else {
            mu = s1 / n;
            float s3 = 0.0f;
#pragma unroll 1
            for (int k = 0; k < 8; k++) {
                float p3 = 0.0f;
#pragma unroll
                for (int i = 0; i < ADD_NORM_CHUNKS; i++) {
                    const int c4 = lane + 32 * k + 256 * i;
                    if (c4 < nc4) {
                        const float4 a = reload_s(c4);
                        const float dx = a.x - mu, dy = a.y - mu, dz = a.z - mu, dw = a.w - mu;
                        p3 = fmaf(dx, dx, fmaf(dy, dy, fmaf(dz, dz, fmaf(dw, dw, p3))));
                    }
                }
                s3 += xor_sum(p3);
            }
            inv = rsqrtf(s3 / n + eps);
        }
        // pass B: bf16 normalised row into shared memory; iteration it covers
        // columns [128 it, 128 it + 128) = quantization block it
#pragma unroll 1
        for (int it = 0; it < nb; it++) {
            const int c4 = it * 32 + lane;
            const float4 a = reload_s(c4);
            const float4 gg = reinterpret_cast<const float4 *>(g)[c4];
            float4 o;
            o.x = (a.x - mu) * inv * gg.x; o.y = (a.y - mu) * inv * gg.y;
            o.z = (a.z - mu) * inv * gg.z; o.w = (a.w - mu) * inv * gg.w;
            if (MODE == 1) {
                const float4 bb = reinterpret_cast<const float4 *>(b)[c4];
                o.x += bb.x; o.y += bb.y; o.z += bb.z; o.w += bb.w;
            }
            const __nv_bfloat162 p0 = __floats2bfloat162_rn(o.x, o.y), p1 = __floats2bfloat162_rn(o.z, o.w);
            uint2 wv;
            wv.x = *reinterpret_cast<const uint32_t *>(&p0);
            wv.y = *reinterpret_cast<const uint32_t *>(&p1);
            reinterpret_cast<uint2 *>(a_s + (size_t)warp * cols)[c4] = wv;
            const float2 f0 = __bfloat1622float2(p0), f1 = __bfloat1622float2(p1);
            float m = fmaxf(fmaxf(fabsf(f0.x), fabsf(f0.y)), fmaxf(fabsf(f1.x), fabsf(f1.y)));
            m = warp_max<32>(m);
            if (lane == 0) amax[warp * nb + it] = m;
        }
    } else {
        for (int it = lane; it < nb; it += 32) amax[warp * nb + it] = 0.0f;   // padding rows of the last band
    }
    __syncthreads();
    for (int t = threadIdx.x; t < nb; t += blockDim.x) {
        float m = 0.0f;
#pragma unroll
        for (int r = 0; r < ANQ_ROWS; r++) m = fmaxf(m, amax[r * nb + t]);
        bmax[t] = m;
    }
    // the band's block maxima over the 8 CTAs of the cluster (DSMEM)
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    for (int t = threadIdx.x; t < nb; t += blockDim.x) {
        float m = 0.0f;
        const uint32_t local = (uint32_t)__cvta_generic_to_shared(bmax + t);
#pragma unroll
        for (int r = 0; r < ANQ_CLUSTER; r++) {
            uint32_t remote;
            float v;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(r));
            asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(remote) : "memory");
            m = fmaxf(m, v);
        }
        const float sc = quant_scale(m);
        bsc[t] = sc;
        if (rank == 0) scales[band * nb + t] = sc;
    }
    __syncthreads();
    if (ok) {
        // pass C: codes from shared memory (quantize_blockwise rule, blockquant.py:106-109)
#pragma unroll 1
        for (int it = 0; it < nb; it++) {
            const float sc = bsc[it];
            const float safe = (sc == 0.0f) ? 1.0f : sc;
            const float rq = __frcp_rn(safe);
            const bool exq = !(safe >= 1.17549435e-38f && rq <= 3.0e38f);   // subnormal scale: exact division
            const int c4 = it * 32 + lane;
            const uint2 wv = reinterpret_cast<const uint2 *>(a_s + (size_t)warp * cols)[c4];
            const float2 f0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&wv.x));
            const float2 f1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&wv.y));
            const float v4[4] = {f0.x, f0.y, f1.x, f1.y};
            uint32_t w[1];
            quant_fast_n<4>(v4, safe, rq, exq, w);
            reinterpret_cast<uint32_t *>(q + row * cols)[c4] = w[0];
        }
    }
    // no CTA leaves while a peer may still read its block maxima
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Instrumentation (tools/step_ablate.py): the %globaltimer value when this
// one-thread kernel runs on its stream -- usable inside CUDA graphs, where
// event timing is not.
__global__ void timestamp_kernel(unsigned long long *dst) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    *dst = t;
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

extern "C" int tb_linear_operands(const void *q, const void *k, const void *v, int dtype, int64_t H, int64_t L,
                                  int64_t d, int64_t lq, int64_t lk, int64_t dx, void *phiq, void *phik, void *vext,
                                  int out_dtype, void *vt, int64_t lvt, void *stream) {
    TB_REQUIRE(d % 8 == 0 && d <= 256, "head_dim must be a multiple of 8 (<= 256)");
    TB_REQUIRE(!phik || (vext && dx >= d + 1 && dx % 8 == 0), "vext needs dx >= d+1, dx % 8 == 0");
    TB_REQUIRE((!phiq || lq >= L) && (!phik || lk >= L) && (!vt || lvt >= L), "padded lengths must cover L");
    TB_REQUIRE(!vt || lvt % 8 == 0, "lvt must be a multiple of 8");
    if (H == 0) return TB_OK;
    int64_t lmax = 0;
    if (phiq && lq > lmax) lmax = lq;
    if (phik && lk > lmax) lmax = lk;
    if (vt && lvt > lmax) lmax = lvt;
    if (lmax == 0) return TB_OK;
    const int cg = (int)(d / 8);
    const int threads = (256 / cg) * cg;
    dim3 grid((unsigned)cdiv(lmax, 64), (unsigned)H);
    const size_t smem = vt ? (size_t)64 * (d + 2) * 2 : 0;
    cudaStream_t st = as_stream(stream);
#define TB_LINOP(T, O)                                                                                           \
    linear_operands_kernel<T, O><<<grid, threads, smem, st>>>((const T *)q, (const T *)k, (const T *)v, L, (int)d, \
                                                              lq, lk, (int)dx, (O *)phiq, (O *)phik, (O *)vext,  \
                                                              (__nv_bfloat16 *)vt, lvt)
    if (dtype == TB_F32 && out_dtype == TB_BF16) TB_LINOP(float, __nv_bfloat16);
    else if (dtype == TB_F32) TB_LINOP(float, float);
    else if (out_dtype == TB_BF16) TB_LINOP(__nv_bfloat16, __nv_bfloat16);
    else TB_LINOP(__nv_bfloat16, float);
#undef TB_LINOP
    return check_launch("linear_operands");
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

extern "C" int tb_timestamp(unsigned long long *dst, void *stream) {
    timestamp_kernel<<<1, 1, 0, as_stream(stream)>>>(dst);
    return check_launch("timestamp");
}

extern "C" int tb_add_norm(const float *x, const float *y, const float *emb, float alpha, const float *gain,
                           const float *offset, int64_t rows, int64_t cols, float eps, int layer_norm,
                           float *sum_out, void *norm_out, void *stream) {
    TB_REQUIRE(eps > 0.0f, "eps must be > 0");
    TB_REQUIRE(cols % 4 == 0 && cols <= 4 * 256 * ADD_NORM_CHUNKS, "cols must be a multiple of 4, <= 8192");
    TB_REQUIRE(!layer_norm || offset != nullptr, "layer norm needs an offset");
    if (rows == 0) return TB_OK;
    cudaStream_t st = as_stream(stream);
    if (layer_norm)
        add_norm_kernel<1><<<(unsigned)rows, 256, 0, st>>>(x, y, emb, alpha, gain, offset, cols, eps, sum_out,
                                                          (__nv_bfloat16 *)norm_out);
    else
        add_norm_kernel<0><<<(unsigned)rows, 256, 0, st>>>(x, y, emb, alpha, gain, offset, cols, eps, sum_out,
                                                          (__nv_bfloat16 *)norm_out);
    return check_launch("add_norm");
}

// add_norm + block-128 quantization of the normalised (bf16-rounded) rows in
// one kernel: codes [rows, cols] int8 + scales [ceil(rows/128), cols/128] f32,
// bit-identical to tb_add_norm (norm_out) followed by tb_quantize_blockwise
// (block 128).  cols % 128 == 0, cols <= 6144.
extern "C" int tb_add_norm_quant(const float *x, const float *y, const float *emb, float alpha, const float *gain,
                                 const float *offset, int64_t rows, int64_t cols, float eps, int layer_norm,
                                 float *sum_out, int8_t *q, float *scales, void *stream) {
    TB_REQUIRE(eps > 0.0f, "eps must be > 0");
    TB_REQUIRE(cols % 128 == 0 && cols >= 128 && cols <= 6144, "cols must be a multiple of 128, <= 6144");
    TB_REQUIRE(!layer_norm || offset != nullptr, "layer norm needs an offset");
    TB_REQUIRE(((uintptr_t)x % 16) == 0 && ((uintptr_t)q % 4) == 0 && (y == nullptr || (uintptr_t)y % 16 == 0) &&
                   (sum_out == nullptr || (uintptr_t)sum_out % 16 == 0),
               "x, y, sum_out must be 16-byte aligned, q 4-byte aligned");
    if (rows == 0) return TB_OK;
    const int nb = (int)(cols / 128);
    const size_t smem = (size_t)ANQ_ROWS * cols * 2 + (size_t)(ANQ_ROWS + 2) * nb * 4;
    const unsigned grid = (unsigned)(cdiv(rows, 128) * ANQ_CLUSTER);
    cudaStream_t st = as_stream(stream);
    if (layer_norm) {
        smem_attr(add_norm_quant_kernel<1>, (int)smem);
        add_norm_quant_kernel<1><<<grid, ANQ_ROWS * 32, smem, st>>>(x, y, emb, alpha, gain, offset, rows, (int)cols,
                                                                     eps, sum_out, q, scales);
    } else {
        smem_attr(add_norm_quant_kernel<0>, (int)smem);
        add_norm_quant_kernel<0><<<grid, ANQ_ROWS * 32, smem, st>>>(x, y, emb, alpha, gain, offset, rows, (int)cols,
                                                                     eps, sum_out, q, scales);
    }
    return check_launch("add_norm_quant");
}

// ------------------------------------------------------------ delta merging
// merge.py apply_deltas (merge.py:55-71): merged = merged + f32(c) * delta in
// list order, numpy's two roundings (RN multiply, then RN add; no FMA).
__global__ void axpy_rn_kernel(float *__restrict__ acc, const float *__restrict__ x, float c, int64_t n) {
    const int64_t n4 = n >> 2;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
        float4 a = reinterpret_cast<float4 *>(acc)[i];
        const float4 d = __ldg(reinterpret_cast<const float4 *>(x) + i);
        a.x = __fadd_rn(a.x, __fmul_rn(c, d.x));
        a.y = __fadd_rn(a.y, __fmul_rn(c, d.y));
        a.z = __fadd_rn(a.z, __fmul_rn(c, d.z));
        a.w = __fadd_rn(a.w, __fmul_rn(c, d.w));
        reinterpret_cast<float4 *>(acc)[i] = a;
    }
    for (int64_t i = 4 * n4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        acc[i] = __fadd_rn(acc[i], __fmul_rn(c, x[i]));
}

extern "C" int tb_axpy_rn(float *acc, const float *x, float c, int64_t n, void *stream) {
    TB_REQUIRE(((uintptr_t)acc & 15) == 0 && ((uintptr_t)x & 15) == 0, "acc and x must be 16-byte aligned");
    if (n == 0) return TB_OK;
    const int64_t blocks = imin64(cdiv(cdiv(n, 4), 256), 148 * 8);
    axpy_rn_kernel<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(acc, x, c, n);
    return check_launch("axpy_rn");
}

// f32 -> bf16 (RN) copy: the bf16 V operand (tb_sla_args.vt) of the
// tensor-core attention kernel when the inputs are f32 (the drop-in's numpy
// path).  8 elements per thread, 16-B stores.
__global__ void cast_bf16_kernel(const float *__restrict__ x, __nv_bfloat16 *__restrict__ y, int64_t n) {
    const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 8;
    if (i + 8 <= n) {
        const float4 a = *reinterpret_cast<const float4 *>(x + i), b = *reinterpret_cast<const float4 *>(x + i + 4);
        uint4 w;
        __nv_bfloat162 *p = reinterpret_cast<__nv_bfloat162 *>(&w);
        p[0] = __floats2bfloat162_rn(a.x, a.y);
        p[1] = __floats2bfloat162_rn(a.z, a.w);
        p[2] = __floats2bfloat162_rn(b.x, b.y);
        p[3] = __floats2bfloat162_rn(b.z, b.w);
        *reinterpret_cast<uint4 *>(y + i) = w;
    } else {
        for (int64_t j = i; j < n; j++) y[j] = __float2bfloat16_rn(x[j]);
    }
}

extern "C" int tb_cast_bf16(const float *x, int64_t n, void *y, void *stream) {
    TB_REQUIRE(((uintptr_t)x & 15) == 0 && ((uintptr_t)y & 15) == 0, "x and y must be 16-byte aligned");
    if (n == 0) return TB_OK;
    cast_bf16_kernel<<<(unsigned)cdiv(cdiv(n, 8), 256), 256, 0, as_stream(stream)>>>(
        x, reinterpret_cast<__nv_bfloat16 *>(y), n);
    return check_launch("cast_bf16");
}

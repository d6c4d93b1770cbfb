// quant.cu -- bit-exact block quantization, pooling and k_mean kernels (HBM-bound).
//
// Replaces (reference /root/reference/pkg/src/turbobench/):
//   blockquant.quantize_blockwise      blockquant.py:91-110
//   blockquant.dequantize_blockwise    blockquant.py:113-116
//   attention.pool_block_means         attention.py:256-266
//   attention.smooth_keys (k_mean)     attention.py:179-188
//   attention._quantize_token_blocks   attention.py:201-220
#include "common.cuh"
#include "ptx.cuh"
#include "tmap.cuh"

namespace tb {

// ---------------------------------------------------- quantize_blockwise
// One CTA per (block x block) tile.  Pass 1: absmax (order-free) + finite
// check; pass 2 re-reads the tile (L1/L2 hit) and writes codes.
template <typename T>
__global__ void __launch_bounds__(256) quantize_blockwise_kernel(
    const T *__restrict__ x, int64_t rows, int64_t cols, int64_t block, int64_t nbc,
    int8_t *__restrict__ q, float *__restrict__ scales, int32_t *__restrict__ nonfinite) {
    __shared__ float red[32];
    const int64_t bi = blockIdx.y, bj = blockIdx.x;
    const int64_t r0 = bi * block, c0 = bj * block;
    const int64_t nr = min(block, rows - r0), nc = min(block, cols - c0);
    const int64_t n = nr * nc;
    float am = 0.0f;
    bool bad = false;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        int64_t r = i / nc, c = i - r * nc;
        float v = to_f32(x[(r0 + r) * cols + c0 + c]);
        bad |= !isfinite(v);
        am = fmaxf(am, fabsf(v));
    }
    if (nonfinite && __syncthreads_or(bad) && threadIdx.x == 0) atomicOr(nonfinite, 1);
    am = block_max_nonneg(am, red);
    const float s = quant_scale(am);
    if (threadIdx.x == 0) scales[bi * nbc + bj] = s;
    const float safe = (s == 0.0f) ? 1.0f : s;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        int64_t r = i / nc, c = i - r * nc;
        q[(r0 + r) * cols + c0 + c] = quant_code(to_f32(x[(r0 + r) * cols + c0 + c]), safe);
    }
}

// Fast path: block == 128, cols % 8 == 0.  Each thread owns 8 consecutive
// columns of a row (16 B of bf16 / 32 B of f32 loaded as vectors), codes
// stored as one 8-byte word.
// PLANAR: x is stored as cols/128 planes [rows, 128] (a head-major attention
// output [H, L, head_dim]); codes and scales are written for the logical
// [rows, cols] matrix (the out-projection's A operand).
template <typename T, bool PLANAR = false>
__global__ void __launch_bounds__(256, sizeof(T) == 2 ? 3 : 2) quantize_blockwise128_kernel(
    const T *__restrict__ x, int64_t rows, int64_t cols, int64_t nbc,
    int8_t *__restrict__ q, float *__restrict__ scales, int32_t *__restrict__ nonfinite) {
    __shared__ float red[32];
    const int64_t bi = blockIdx.y, bj = blockIdx.x;
    const int64_t r0 = bi * 128, c0 = bj * 128;
    const int nr = (int)imin64(128, rows - r0), nc = (int)imin64(128, cols - c0);
    const int lane16 = threadIdx.x & 15;           // column group (8 cols each)
    const int rsub = threadIdx.x >> 4;             // 16 rows per pass
    const bool col_ok = lane16 * 8 < nc;
    // bf16 input stays packed in registers (32 instead of 64), so 4 CTAs fit
    // per SM and 128 KB of loads are in flight per SM; unpacked on use
    constexpr bool PACKED = sizeof(T) == 2;
    float v[PACKED ? 1 : 8][8];
    uint4 raw[PACKED ? 8 : 1];
    auto unpack = [&](int p, float (&f)[8]) {
        const __nv_bfloat162 *b = reinterpret_cast<const __nv_bfloat162 *>(&raw[PACKED ? p : 0]);
#pragma unroll
        for (int j = 0; j < 4; j++) { const float2 t = __bfloat1622float2(b[j]); f[2 * j] = t.x; f[2 * j + 1] = t.y; }
    };
    float am = 0.0f;
    bool bad = false;
#pragma unroll
    for (int p = 0; p < 8; p++) {
        int r = rsub + p * 16;
        if constexpr (PACKED) raw[p] = make_uint4(0u, 0u, 0u, 0u);
        if (col_ok && r < nr) {
            const T *src = PLANAR ? x + (c0 / 128) * rows * 128 + (r0 + r) * 128 + lane16 * 8
                                  : x + (r0 + r) * cols + c0 + lane16 * 8;
            if constexpr (PACKED) raw[p] = __ldg(reinterpret_cast<const uint4 *>(src));
        }
    }
#pragma unroll
    for (int p = 0; p < 8; p++) {
        int r = rsub + p * 16;
        if (col_ok && r < nr) {
            const T *src = PLANAR ? x + (c0 / 128) * rows * 128 + (r0 + r) * 128 + lane16 * 8
                                  : x + (r0 + r) * cols + c0 + lane16 * 8;
            float vv[8];
            if constexpr (PACKED) {
                unpack(p, vv);
#pragma unroll
                for (int j = 0; j < 8; j++) {
                    bad |= !isfinite(vv[j]);
                    am = fmaxf(am, fabsf(vv[j]));
                }
                continue;
            } else {
                float4 a = *reinterpret_cast<const float4 *>(src);
                float4 b = *reinterpret_cast<const float4 *>(src + 4);
                v[p][0] = a.x; v[p][1] = a.y; v[p][2] = a.z; v[p][3] = a.w;
                v[p][4] = b.x; v[p][5] = b.y; v[p][6] = b.z; v[p][7] = b.w;
            }
#pragma unroll
            for (int j = 0; j < 8; j++) {
                bad |= !isfinite(v[p][j]);
                am = fmaxf(am, fabsf(v[p][j]));
            }
        }
    }
    if (nonfinite && __syncthreads_or(bad) && threadIdx.x == 0) atomicOr(nonfinite, 1);
    am = block_max_nonneg(am, red);
    const float s = quant_scale(am);
    if (threadIdx.x == 0) scales[bi * nbc + bj] = s;
    const float safe = (s == 0.0f) ? 1.0f : s;
    const float inv = __frcp_rn(safe);
    const bool exact = !(safe >= 1.17549435e-38f && inv <= 3.0e38f);   // subnormal scale: exact division
#pragma unroll
    for (int p = 0; p < 8; p++) {
        int r = rsub + p * 16;
        if (col_ok && r < nr) {
            // branch-free fast codes (bit-identical; near-ties redone exactly)
            float vq[8];
            if constexpr (PACKED) {
                unpack(p, vq);
            } else {
#pragma unroll
                for (int j = 0; j < 8; j++) vq[j] = v[p][j];
            }
            uint32_t w[2];
            quant_fast_n<8>(vq, safe, inv, exact, w);
            *reinterpret_cast<uint2 *>(q + (r0 + r) * cols + c0 + lane16 * 8) = make_uint2(w[0], w[1]);
        }
    }
}

__global__ void dequantize_blockwise_kernel(const int8_t *__restrict__ q, const float *__restrict__ scales,
                                            int64_t rows, int64_t cols, int64_t block, int64_t nbc,
                                            float *__restrict__ out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= rows * cols) return;
    int64_t r = i / cols, c = i - r * cols;
    out[i] = (float)q[i] * scales[(r / block) * nbc + c / block];
}

__global__ void transpose_codes_kernel(const int8_t *__restrict__ src, int64_t rows, int64_t cols,
                                       int8_t *__restrict__ dst) {
    __shared__ int8_t tile[32][33];
    int64_t c = blockIdx.x * 32 + threadIdx.x, r = blockIdx.y * 32 + threadIdx.y;
    for (int k = 0; k < 32; k += 8)
        if (r + k < rows && c < cols) tile[threadIdx.y + k][threadIdx.x] = src[(r + k) * cols + c];
    __syncthreads();
    int64_t oc = blockIdx.y * 32 + threadIdx.x, orow = blockIdx.x * 32 + threadIdx.y;
    for (int k = 0; k < 32; k += 8)
        if (orow + k < cols && oc < rows) dst[(orow + k) * rows + oc] = tile[threadIdx.x][threadIdx.y + k];
}

// --------------------------------------------------------- pooling order
// numpy pairwise summation (FLOAT_pairwise_sum, PW_BLOCKSIZE 128) over n
// elements at `stride`, in f32.
template <typename T>
__device__ float pw_sum(const T *a, int64_t n, int64_t stride) {
    if (n < 8) {
        float res = -0.0f;
        for (int64_t i = 0; i < n; i++) res = __fadd_rn(res, to_f32(a[i * stride]));
        return res;
    } else if (n <= 128) {
        float r[8];
#pragma unroll
        for (int j = 0; j < 8; j++) r[j] = to_f32(a[j * stride]);
        int64_t i;
        for (i = 8; i < n - (n % 8); i += 8) {
#pragma unroll
            for (int j = 0; j < 8; j++) r[j] = __fadd_rn(r[j], to_f32(a[(i + j) * stride]));
        }
        float res = __fadd_rn(__fadd_rn(__fadd_rn(r[0], r[1]), __fadd_rn(r[2], r[3])),
                              __fadd_rn(__fadd_rn(r[4], r[5]), __fadd_rn(r[6], r[7])));
        for (; i < n; i++) res = __fadd_rn(res, to_f32(a[i * stride]));
        return res;
    } else {
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        return __fadd_rn(pw_sum(a, n2, stride), pw_sum(a + n2 * stride, n - n2, stride));
    }
}

// --------------------------------------------------- token-block pool+quant
// One CTA per (head, token block).  Thread per channel (strided if d >
// blockDim): pooled mean of the raw x in numpy reduceat order, absmax of
// (x - center), then codes of (x - center).
template <typename T>
__global__ void __launch_bounds__(128) pool_quant_tokens_kernel(
    const T *__restrict__ x, const float *__restrict__ center, int64_t L, int64_t d, int64_t block,
    int64_t nb, int8_t *__restrict__ codes, float *__restrict__ scales, float *__restrict__ pooled) {
    __shared__ float red[32];
    const int64_t h = blockIdx.y, b = blockIdx.x;
    const int64_t lo = b * block, e = min(block, L - lo);
    const T *xb = x + (h * L + lo) * d;
    float am = 0.0f;
    for (int64_t c = threadIdx.x; c < d; c += blockDim.x) {
        const float ctr = center ? center[h * d + c] : 0.0f;
        if (pooled) {
            float acc = to_f32(xb[c]);
            if (e > 1) acc = __fadd_rn(acc, pw_sum(xb + d + c, e - 1, d));
            pooled[(h * nb + b) * d + c] = __fdiv_rn(acc, (float)e);
        }
        if (codes) {
            for (int64_t t = 0; t < e; t++) {
                float v = center ? __fsub_rn(to_f32(xb[t * d + c]), ctr) : to_f32(xb[t * d + c]);
                am = fmaxf(am, fabsf(v));
            }
        }
    }
    if (!codes) return;
    am = block_max_nonneg(am, red);
    const float s = quant_scale(am);
    if (threadIdx.x == 0) scales[h * nb + b] = s;
    const float safe = (s == 0.0f) ? 1.0f : s;
    int8_t *cb = codes + (h * L + lo) * d;
    for (int64_t i = threadIdx.x; i < e * d; i += blockDim.x) {
        int64_t c = i % d;
        float v = to_f32(xb[i]);
        if (center) v = __fsub_rn(v, center[h * d + c]);
        cb[i] = quant_code(v, safe);
    }
}

// Fast path for d == 128, block <= 129 (the hot-path shapes): 128 threads,
// thread c owns channel c.  Pass 1 streams the tile once in token order,
// computing the numpy reduceat pooled sum (seed + pairwise of the rest, the
// 8-accumulator body of FLOAT_pairwise_sum consumed as the values arrive) and
// the absmax; pass 2 re-reads the (L1-resident) tile for the codes, which are
// transposed through shared memory so each warp stores contiguous 128 B rows.
template <typename T, int BLOCK>
__global__ void __launch_bounds__(128) pool_quant_tokens_d128_kernel(
    const T *__restrict__ x, const float *__restrict__ center, int64_t L, int64_t nb,
    int8_t *__restrict__ codes, float *__restrict__ scales, float *__restrict__ pooled) {
    __shared__ float red[32];
    __shared__ __align__(16) int8_t stile[BLOCK][128];
    const int64_t h = blockIdx.y, b = blockIdx.x;
    const int64_t lo = b * BLOCK;
    const int e = (int)imin64(BLOCK, L - lo);
    const int c = threadIdx.x;
    const T *xb = x + (h * L + lo) * 128 + c;
    const float ctr = center ? center[h * 128 + c] : 0.0f;
    auto ld = [&](int t) { return to_f32(xb[(int64_t)t * 128]); };
    float am = 0.0f;
    const float seed = ld(0);
    am = fabsf(seed - ctr);
    const int n = e - 1;                               // values after the seed
    float res = -0.0f;
    if (n >= 8) {
        float r[8];
#pragma unroll
        for (int j = 0; j < 8; j++) { r[j] = ld(1 + j); am = fmaxf(am, fabsf(r[j] - ctr)); }
        const int full = n - (n % 8);
        for (int i = 8; i < full; i += 8) {
            float w[8];
#pragma unroll
            for (int j = 0; j < 8; j++) w[j] = ld(1 + i + j);
#pragma unroll
            for (int j = 0; j < 8; j++) { r[j] = __fadd_rn(r[j], w[j]); am = fmaxf(am, fabsf(w[j] - ctr)); }
        }
        res = __fadd_rn(__fadd_rn(__fadd_rn(r[0], r[1]), __fadd_rn(r[2], r[3])),
                        __fadd_rn(__fadd_rn(r[4], r[5]), __fadd_rn(r[6], r[7])));
        for (int i = full; i < n; i++) { const float w = ld(1 + i); res = __fadd_rn(res, w); am = fmaxf(am, fabsf(w - ctr)); }
    } else {
        for (int i = 0; i < n; i++) { const float w = ld(1 + i); res = __fadd_rn(res, w); am = fmaxf(am, fabsf(w - ctr)); }
    }
    if (pooled) {
        const float acc = (n > 0) ? __fadd_rn(seed, res) : seed;
        pooled[(h * nb + b) * 128 + c] = __fdiv_rn(acc, (float)e);
    }
    am = block_max_nonneg(am, red);
    const float s = quant_scale(am);
    if (threadIdx.x == 0) scales[h * nb + b] = s;
    const float safe = (s == 0.0f) ? 1.0f : s;
    for (int t0 = 0; t0 < e; t0 += 8) {
        float w[8];
#pragma unroll
        for (int j = 0; j < 8; j++) w[j] = (t0 + j < e) ? ld(t0 + j) : 0.0f;
#pragma unroll
        for (int j = 0; j < 8; j++)
            if (t0 + j < e) stile[t0 + j][c] = quant_code(center ? __fsub_rn(w[j], ctr) : w[j], safe);
    }
    __syncthreads();
    int8_t *cb = codes + (h * L + lo) * 128;
    const uint4 *st = reinterpret_cast<const uint4 *>(&stile[0][0]);
    for (int i = threadIdx.x; i < e * 8; i += 128) reinterpret_cast<uint4 *>(cb)[i] = st[i];
}

// five CTAs per SM (48 registers, a few bytes of spill): 15-20% faster Q pass,
// K codes and K pool than the 64-register, four-CTA build (tools/time_poolq.py,
// interleaved A/B) -- more tiles' bulk loads in flight per SM
#ifndef TB_POOLQ_MINB
#define TB_POOLQ_MINB 5
#endif
// Tile kernel for bf16 inputs, d == 128, block 64 or 128 (the hot path):
// one CTA per 128-token tile of one head (one Q block of 128 or two K blocks
// of 64), 256 threads.  The 32 KB tile arrives in shared memory with one bulk
// copy and is read twice from there:
//   pass 1 (all threads: channel pair x a share of the 8 pairwise
//          accumulators): numpy's reduceat order for the pooled sum (seed +
//          8-accumulator pairwise body + sequential tail, both channels in
//          f32x2 lanes) and the absmax of the (centered) values
//   pass 2 (all threads, 16 channels x one token each): codes via
//          quant_code_fast (bit-exact with the IEEE division), 16-B stores.
template <int BLOCK>
__global__ void __launch_bounds__(256, TB_POOLQ_MINB) pool_quant_tile_kernel(
    const __nv_bfloat16 *__restrict__ x, const float *__restrict__ center, int64_t L, int64_t nb,
    int8_t *__restrict__ codes, float *__restrict__ scales, float *__restrict__ pooled,
    float *__restrict__ pooled_t, int64_t ldt) {
    constexpr int TT = 128, NBLK = TT / BLOCK;
    __shared__ __align__(128) __nv_bfloat16 tile[TT * 128];
    __shared__ __align__(8) uint64_t full;
    __shared__ float red[NBLK][2 * (256 / (64 * NBLK))];   // per warp: absmax of its values
    __shared__ float2 part[NBLK][256 / (64 * NBLK)][64];    // per sub: its pairwise subtree
    __shared__ float bsafe[NBLK], binv[NBLK];
    __shared__ int bexact[NBLK];
    const int64_t h = blockIdx.y;
    const int64_t lo = (int64_t)blockIdx.x * TT;
    const int et = (int)imin64(TT, L - lo);                    // tokens in this tile
    if (threadIdx.x == 0) {
        ptx::mbar_init(&full, 1);
        ptx::fence_barrier_init();
        ptx::mbar_arrive_expect_tx(&full, (uint32_t)et * 256u);
        ptx::bulk_g2s(tile, x + (h * L + lo) * 128, (uint32_t)et * 256u, &full);
    }
    __syncthreads();
    ptx::mbar_wait(&full, 0);
    const int tid = threadIdx.x;
    // ---- pass 1: pooled sums (raw x) + absmax (centered).  Thread = (block,
    // channel pair, sub): a full block's 8 pairwise accumulators are split over
    // SUBS threads (independent chains, combined below in numpy's tree order);
    // a ragged last block runs the whole order on its sub-0 thread.  A warp is
    // 32 channel pairs of one (block, sub): conflict-free shared-memory reads.
    constexpr int SUBS = 256 / (64 * NBLK), JPS = 8 / SUBS;
    const int cp = tid & 63, grp = tid >> 6, blk = grp % NBLK, sub = grp / NBLK;
    const int t0 = blk * BLOCK;
    const int e = min(BLOCK, et - t0);
    const bool whole = e == BLOCK;                           // uniform per warp
    const float2 ctr = center ? *reinterpret_cast<const float2 *>(center + h * 128 + 2 * cp) : make_float2(0.0f, 0.0f);
    const uint32_t *col = reinterpret_cast<const uint32_t *>(tile) + cp;   // row stride 64 words
    auto ld = [&](int t) {
        const uint32_t w = col[(t0 + t) * 64];
        return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xFFFF0000u));
    };
    float am0 = 0.0f, am1 = 0.0f;
    auto amax = [&](float2 v) {
        am0 = fmaxf(am0, fabsf(__fsub_rn(v.x, ctr.x)));
        am1 = fmaxf(am1, fabsf(__fsub_rn(v.y, ctr.y)));
    };
    auto store_pool = [&](float2 acc, int cnt) {
        const int64_t b = lo / BLOCK + blk;
        const float2 pm = make_float2(__fdiv_rn(acc.x, (float)cnt), __fdiv_rn(acc.y, (float)cnt));
        *reinterpret_cast<float2 *>(pooled + (h * nb + b) * 128 + 2 * cp) = pm;
        if (pooled_t) {                                      // [H][d][ldt] copy: the top-k kernel's coalesced operand
            pooled_t[(h * 128 + 2 * cp) * ldt + b] = pm.x;
            pooled_t[(h * 128 + 2 * cp + 1) * ldt + b] = pm.y;
        }
    };
    // full block: n = BLOCK - 1 elements after the seed, body i < FULL8 in 8 chains, tail FULL8..n-1
    constexpr int N1 = BLOCK - 1, FULL8 = N1 - N1 % 8;
    if (whole) {
        float2 r[JPS];
#pragma unroll
        for (int u = 0; u < JPS; u++) { r[u] = ld(1 + sub * JPS + u); amax(r[u]); }
#pragma unroll 4
        for (int i = 8; i < FULL8; i += 8) {
#pragma unroll
            for (int u = 0; u < JPS; u++) { const float2 w = ld(1 + i + sub * JPS + u); r[u] = ptx::fadd2(r[u], w); amax(w); }
        }
        // this thread's subtree of ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7))
        float2 p = ptx::fadd2(r[0], r[1]);
        if constexpr (JPS == 4) p = ptx::fadd2(p, ptx::fadd2(r[2], r[3]));
        part[blk][sub][cp] = p;
        if (sub == 0) {
            amax(ld(0));
#pragma unroll
            for (int i = FULL8; i < N1; i++) amax(ld(1 + i));
        }
    } else if (sub == 0 && e > 0) {
        const float2 seed = ld(0);
        amax(seed);
        const int n = e - 1;
        float2 res = make_float2(-0.0f, -0.0f);
        if (n >= 8) {
            float2 r[8];
#pragma unroll
            for (int j = 0; j < 8; j++) { r[j] = ld(1 + j); amax(r[j]); }
            const int full8 = n - (n % 8);
            for (int i = 8; i < full8; i += 8) {
#pragma unroll
                for (int j = 0; j < 8; j++) { const float2 w = ld(1 + i + j); r[j] = ptx::fadd2(r[j], w); amax(w); }
            }
            res = ptx::fadd2(ptx::fadd2(ptx::fadd2(r[0], r[1]), ptx::fadd2(r[2], r[3])),
                             ptx::fadd2(ptx::fadd2(r[4], r[5]), ptx::fadd2(r[6], r[7])));
            for (int i = full8; i < n; i++) { const float2 w = ld(1 + i); res = ptx::fadd2(res, w); amax(w); }
        } else {
            for (int i = 0; i < n; i++) { const float2 w = ld(1 + i); res = ptx::fadd2(res, w); amax(w); }
        }
        if (pooled) store_pool((n > 0) ? ptx::fadd2(seed, res) : seed, e);
    }
    {
        float am = fmaxf(am0, am1);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) am = fmaxf(am, __shfl_xor_sync(0xffffffffu, am, o));
        if ((tid & 31) == 0) red[blk][sub * 2 + ((tid >> 5) & 1)] = am;
    }
    __syncthreads();
    if (whole && sub == 0 && pooled) {
        float2 res = ptx::fadd2(part[blk][0][cp], part[blk][1][cp]);
        if constexpr (SUBS == 4) res = ptx::fadd2(res, ptx::fadd2(part[blk][2][cp], part[blk][3][cp]));
#pragma unroll
        for (int i = FULL8; i < N1; i++) res = ptx::fadd2(res, ld(1 + i));
        store_pool(ptx::fadd2(ld(0), res), BLOCK);
    }
    if (codes == nullptr) return;                            // pooling only (uniform)
    if (tid < NBLK && tid * BLOCK < et) {
        float am = red[tid][0];
#pragma unroll
        for (int i = 1; i < 2 * SUBS; i++) am = fmaxf(am, red[tid][i]);
        const float s = quant_scale(am);
        scales[h * nb + lo / BLOCK + tid] = s;
        const float safe = (s == 0.0f) ? 1.0f : s;
        const float inv = __frcp_rn(safe);
        bsafe[tid] = safe;
        binv[tid] = inv;
        bexact[tid] = !(safe >= 1.17549435e-38f && inv <= 3.0e38f);   // subnormal scale: exact division
    }
    __syncthreads();
    // ---- pass 2: codes, 16 channels of one token per work item
    const int g = tid & 7;                                   // 16-channel group
    float cg[16];
#pragma unroll
    for (int i = 0; i < 16; i++) cg[i] = center ? __ldg(center + h * 128 + 16 * g + i) : 0.0f;
    for (int t = tid >> 3; t < et; t += 32) {
        const int blk = t / BLOCK;
        const float safe = bsafe[blk], inv = binv[blk];
        const bool exact = bexact[blk] != 0;
        const uint4 *src = reinterpret_cast<const uint4 *>(tile + t * 128 + 16 * g);
        uint32_t wv[8];
        *reinterpret_cast<uint4 *>(&wv[0]) = src[0];
        *reinterpret_cast<uint4 *>(&wv[4]) = src[1];
        float xv[16];
#pragma unroll
        for (int i = 0; i < 16; i++) {
            const uint32_t w = wv[i >> 1];
            float v = __uint_as_float((i & 1) ? (w & 0xFFFF0000u) : (w << 16));
            if (center) v = __fsub_rn(v, cg[i]);
            xv[i] = v;
        }
        uint32_t out[4];
        quant16_fast(xv, safe, inv, exact, out);
        *reinterpret_cast<uint4 *>(codes + (h * L + lo + t) * 128 + 16 * g) = make_uint4(out[0], out[1], out[2], out[3]);
    }
}

// ------------------------------------------------------------------ k_mean
// Sequential f32 chain over all L tokens per (head, channel) -- the numpy
// strided-reduce order.  The chain is latency-bound
// (L dependent FADDs), so the kernel streams the head's [L,d] slab through a
// shared-memory ring with 1-D bulk (TMA) copies: one CTA per head, one thread
// per channel, the copy engine keeps STAGES chunks in flight.
template <typename T, int STAGES>
__global__ void __launch_bounds__(128) kmean_bulk_kernel(const T *__restrict__ k, int64_t L, int d,
                                                         int chunk_tokens, float *__restrict__ kmean) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
    const int64_t h = blockIdx.x;
    const T *src = k + h * L * d;
    const int64_t nchunks = cdiv(L, chunk_tokens);
    const uint32_t chunk_bytes = (uint32_t)(chunk_tokens * d * sizeof(T));
    T *ring = reinterpret_cast<T *>(smem);
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; s++) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], blockDim.x); }
        ptx::fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int64_t i = 0; i < imin64(STAGES, nchunks); i++) {
            int64_t toks = imin64(chunk_tokens, L - i * chunk_tokens);
            uint32_t bytes = (uint32_t)(toks * d * sizeof(T));
            ptx::mbar_arrive_expect_tx(&full[i], bytes);
            ptx::bulk_g2s(ring + (size_t)i * chunk_tokens * d, src + i * chunk_tokens * d, bytes, &full[i]);
        }
    }
    (void)chunk_bytes;
    const int c = threadIdx.x;
    float acc = 0.0f;
    for (int64_t i = 0; i < nchunks; i++) {
        const int s = (int)(i % STAGES);
        const uint32_t par = (uint32_t)((i / STAGES) & 1);
        ptx::mbar_wait(&full[s], par);
        const int64_t toks = imin64(chunk_tokens, L - i * chunk_tokens);
        const T *buf = ring + (size_t)s * chunk_tokens * d;
        if (c < d) {
            int64_t t = 0;
            for (; t + 8 <= toks; t += 8) {
                float w[8];
#pragma unroll
                for (int j = 0; j < 8; j++) w[j] = to_f32(buf[(t + j) * d + c]);
#pragma unroll
                for (int j = 0; j < 8; j++) acc = __fadd_rn(acc, w[j]);
            }
            for (; t < toks; t++) acc = __fadd_rn(acc, to_f32(buf[t * d + c]));
        }
        ptx::mbar_arrive(&empty[s]);
        if (threadIdx.x == 0 && i + STAGES < nchunks) {
            ptx::mbar_wait(&empty[s], par);
            const int64_t j = i + STAGES;
            int64_t tk = imin64(chunk_tokens, L - j * chunk_tokens);
            uint32_t bytes = (uint32_t)(tk * d * sizeof(T));
            ptx::mbar_arrive_expect_tx(&full[s], bytes);
            ptx::bulk_g2s(ring + (size_t)s * chunk_tokens * d, src + j * chunk_tokens * d, bytes, &full[s]);
        }
    }
    if (c < d) kmean[h * d + c] = __fdiv_rn(acc, (float)L);
}

// bf16, d == 128: one warp per (head, 32-channel quarter) so 4*H CTAs stream
// the heads in parallel; a 2-D TMA ring of [256 tokens x 32 channels] tiles
// (16 KB) feeds the chains, each lane one channel, summing in token order; the
// next 16 tokens' shared-memory loads issue under the current 16-add chain.
#ifndef TB_KM_PIPE
#define TB_KM_PIPE 1
#endif
constexpr int KM_CH = 256, KM_STAGES = 6;   // ring depth: up to KM_STAGES, chosen at launch
__global__ void __launch_bounds__(32) kmean_split_kernel(const __grid_constant__ CUtensorMap tm, int64_t L,
                                                         int nst, float *__restrict__ kmean) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t full[KM_STAGES];
    const int qc = blockIdx.x, h = blockIdx.y, lane = threadIdx.x;
    const __nv_bfloat16 *ring = reinterpret_cast<const __nv_bfloat16 *>(smem);
    const int64_t nch = cdiv(L, KM_CH);
    const int64_t row0 = (int64_t)h * L;
    if (lane == 0) {
        for (int s = 0; s < nst; s++) ptx::mbar_init(&full[s], 1);
        ptx::fence_barrier_init();
        for (int64_t i = 0; i < imin64(nst, nch); i++) {
            ptx::mbar_arrive_expect_tx(&full[i], KM_CH * 64);
            ptx::tma_load_2d(smem + i * KM_CH * 64, &tm, qc * 32, (int)(row0 + i * KM_CH), &full[i]);
        }
    }
    __syncwarp();
    float acc = 0.0f;
    for (int64_t i = 0; i < nch; i++) {
        const int s = (int)(i % nst);
        ptx::mbar_wait(&full[s], (uint32_t)((i / nst) & 1));
        const int toks = (int)imin64(KM_CH, L - i * KM_CH);
        const __nv_bfloat16 *buf = ring + (size_t)s * KM_CH * 32 + lane;
        int t = 0;
#if TB_KM_PIPE
        if (toks == KM_CH) {
            // full chunk: the next 16 tokens' loads issue before this batch's adds, so the
            // shared-memory latency hides under the 16-add chain
            __nv_bfloat16 w[16], nx[16];
#pragma unroll
            for (int j = 0; j < 16; j++) w[j] = buf[j * 32];
#pragma unroll 1
            for (t = 0; t < KM_CH - 16; t += 16) {
#pragma unroll
                for (int j = 0; j < 16; j++) nx[j] = buf[(t + 16 + j) * 32];
#pragma unroll
                for (int j = 0; j < 16; j++) acc = __fadd_rn(acc, __bfloat162float(w[j]));
#pragma unroll
                for (int j = 0; j < 16; j++) w[j] = nx[j];
            }
#pragma unroll
            for (int j = 0; j < 16; j++) acc = __fadd_rn(acc, __bfloat162float(w[j]));
            t = KM_CH;
        }
#endif
        for (; t + 16 <= toks; t += 16) {
            float w[16];
#pragma unroll
            for (int j = 0; j < 16; j++) w[j] = __bfloat162float(buf[(t + j) * 32]);
#pragma unroll
            for (int j = 0; j < 16; j++) acc = __fadd_rn(acc, w[j]);
        }
        for (; t < toks; t++) acc = __fadd_rn(acc, __bfloat162float(buf[t * 32]));
        __syncwarp();
        if (lane == 0 && i + nst < nch) {
            ptx::fence_async_smem();          // the warp's reads of stage s before the TMA overwrite
            ptx::mbar_arrive_expect_tx(&full[s], KM_CH * 64);
            ptx::tma_load_2d(smem + s * KM_CH * 64, &tm, qc * 32, (int)(row0 + (i + nst) * KM_CH), &full[s]);
        }
    }
    kmean[h * 128 + qc * 32 + lane] = __fdiv_rn(acc, (float)L);
}

// Generic fallback (unaligned rows / large d): same order, direct loads.
template <typename T>
__global__ void kmean_simple_kernel(const T *__restrict__ k, int64_t H, int64_t L, int64_t d,
                                    float *__restrict__ kmean) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= H * d) return;
    int64_t h = i / d, c = i - h * d;
    const T *p = k + h * L * d + c;
    float acc = 0.0f;
    int64_t t = 0;
    for (; t + 8 <= L; t += 8) {
        float w[8];
#pragma unroll
        for (int j = 0; j < 8; j++) w[j] = to_f32(p[(t + j) * d]);
#pragma unroll
        for (int j = 0; j < 8; j++) acc = __fadd_rn(acc, w[j]);
    }
    for (; t < L; t++) acc = __fadd_rn(acc, to_f32(p[t * d]));
    kmean[i] = __fdiv_rn(acc, (float)L);
}

// ---------------------------------------------------------- V transpose
// V [H,L,d] -> bf16 V^T [H,d,l_pad] with zero padding (K-major B operand of
// the PV MMA: rows = channels, contiguous tokens).
template <typename T>
__global__ void transpose_v_kernel(const T *__restrict__ v, int64_t L, int64_t d, int64_t l_pad,
                                   __nv_bfloat16 *__restrict__ vt) {
    __shared__ float tile[32][33];
    const int64_t h = blockIdx.z;
    const int64_t t0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
    for (int k = threadIdx.y; k < 32; k += 8) {
        int64_t t = t0 + k, c = c0 + threadIdx.x;
        tile[k][threadIdx.x] = (t < L && c < d) ? to_f32(v[(h * L + t) * d + c]) : 0.0f;
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += 8) {
        int64_t c = c0 + k, t = t0 + threadIdx.x;
        if (c < d && t < l_pad) vt[(h * d + c) * l_pad + t] = __float2bfloat16_rn(tile[threadIdx.x][k]);
    }
}

}  // namespace tb

using namespace tb;

extern "C" int tb_quantize_blockwise(const void *x, int dtype, int64_t rows, int64_t cols, int64_t block,
                                     int8_t *q, float *scales, int32_t *nonfinite, void *stream) {
    TB_REQUIRE(block >= 1, "block must be >= 1");
    TB_REQUIRE(rows >= 0 && cols >= 0, "negative shape");
    TB_REQUIRE(dtype == TB_F32 || dtype == TB_BF16, "dtype must be f32 or bf16");
    if (rows == 0 || cols == 0) return TB_OK;
    const int64_t nbr = cdiv(rows, block), nbc = cdiv(cols, block);
    TB_REQUIRE(nbr < 65536, "too many row blocks");
    dim3 grid((unsigned)nbc, (unsigned)nbr);
    cudaStream_t st = as_stream(stream);
    bool fast = block == 128 && cols % 8 == 0 && ((uintptr_t)x % 16) == 0;
    if (dtype == TB_F32) {
        if (fast) quantize_blockwise128_kernel<float><<<grid, 256, 0, st>>>((const float *)x, rows, cols, nbc, q, scales, nonfinite);
        else quantize_blockwise_kernel<float><<<grid, 256, 0, st>>>((const float *)x, rows, cols, block, nbc, q, scales, nonfinite);
    } else {
        if (fast) quantize_blockwise128_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>((const __nv_bfloat16 *)x, rows, cols, nbc, q, scales, nonfinite);
        else quantize_blockwise_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>((const __nv_bfloat16 *)x, rows, cols, block, nbc, q, scales, nonfinite);
    }
    return check_launch("quantize_blockwise");
}

extern "C" int tb_dequantize_blockwise(const int8_t *q, const float *scales, int64_t rows, int64_t cols,
                                       int64_t block, float *out, void *stream) {
    TB_REQUIRE(block >= 1, "block must be >= 1");
    int64_t n = rows * cols;
    if (n == 0) return TB_OK;
    dequantize_blockwise_kernel<<<(unsigned)cdiv(n, 256), 256, 0, as_stream(stream)>>>(
        q, scales, rows, cols, block, cdiv(cols, block), out);
    return check_launch("dequantize_blockwise");
}

extern "C" int tb_transpose_codes(const int8_t *src, int64_t rows, int64_t cols, int8_t *dst, void *stream) {
    if (rows == 0 || cols == 0) return TB_OK;
    dim3 grid((unsigned)cdiv(cols, 32), (unsigned)cdiv(rows, 32));
    transpose_codes_kernel<<<grid, dim3(32, 8), 0, as_stream(stream)>>>(src, rows, cols, dst);
    return check_launch("transpose_codes");
}

extern "C" int tb_pool_block_means(const void *x, int dtype, int64_t H, int64_t L, int64_t d, int64_t block,
                                   float *out, void *stream) {
    return tb_pool_quant_tokens(x, dtype, nullptr, H, L, d, block, nullptr, nullptr, out, stream);
}

static int pool_quant_launch(const void *x, int dtype, const float *center, int64_t H, int64_t L, int64_t d,
                             int64_t block, int8_t *codes, float *scales, float *pooled, float *pooled_t,
                             int64_t ldt, void *stream) {
    TB_REQUIRE(block >= 1, "block must be >= 1");
    TB_REQUIRE(dtype == TB_F32 || dtype == TB_BF16, "dtype must be f32 or bf16");
    TB_REQUIRE((codes == nullptr) == (scales == nullptr), "codes and scales go together");
    if (H == 0 || L == 0 || d == 0) return TB_OK;
    const int64_t nb = cdiv(L, block);
    TB_REQUIRE(H < 65536, "too many heads");
    dim3 grid((unsigned)nb, (unsigned)H);
    cudaStream_t st = as_stream(stream);
    const bool fast = d == 128 && (codes != nullptr || pooled != nullptr) && (block == 64 || block == 128);
    if (fast && dtype == TB_BF16 && ((uintptr_t)x % 16) == 0 && ((uintptr_t)codes % 16) == 0 &&
        (pooled == nullptr || ((uintptr_t)pooled % 8) == 0) && (center == nullptr || ((uintptr_t)center % 8) == 0)) {
        dim3 tgrid((unsigned)cdiv(L, 128), (unsigned)H);
        if (block == 64)
            pool_quant_tile_kernel<64><<<tgrid, 256, 0, st>>>((const __nv_bfloat16 *)x, center, L, nb, codes, scales, pooled,
                                                              pooled_t, ldt);
        else
            pool_quant_tile_kernel<128><<<tgrid, 256, 0, st>>>((const __nv_bfloat16 *)x, center, L, nb, codes, scales, pooled,
                                                               pooled_t, ldt);
        return check_launch("pool_quant_tile");
    }
#define TB_POOLQ(T)                                                                                      \
    if (fast && block == 64)                                                                             \
        pool_quant_tokens_d128_kernel<T, 64><<<grid, 128, 0, st>>>((const T *)x, center, L, nb, codes, scales, pooled); \
    else if (fast)                                                                                       \
        pool_quant_tokens_d128_kernel<T, 128><<<grid, 128, 0, st>>>((const T *)x, center, L, nb, codes, scales, pooled); \
    else                                                                                                 \
        pool_quant_tokens_kernel<T><<<grid, 128, 0, st>>>((const T *)x, center, L, d, block, nb, codes, scales, pooled);
    TB_REQUIRE(pooled_t == nullptr, "the transposed pooled copy needs the bf16 tile path");
    if (dtype == TB_F32) { TB_POOLQ(float) } else { TB_POOLQ(__nv_bfloat16) }
#undef TB_POOLQ
    return check_launch("pool_quant_tokens");
}

extern "C" int tb_pool_quant_tokens(const void *x, int dtype, const float *center, int64_t H, int64_t L,
                                    int64_t d, int64_t block, int8_t *codes, float *scales, float *pooled,
                                    void *stream) {
    return pool_quant_launch(x, dtype, center, H, L, d, block, codes, scales, pooled, nullptr, 0, stream);
}

extern "C" int tb_pool_quant_tokens_t(const void *x, int dtype, const float *center, int64_t H, int64_t L,
                                      int64_t d, int64_t block, int8_t *codes, float *scales, float *pooled,
                                      float *pooled_t, int64_t ldt, void *stream) {
    TB_REQUIRE(pooled != nullptr && pooled_t != nullptr && ldt >= cdiv(L, block), "pooled_t needs ldt >= blocks");
    return pool_quant_launch(x, dtype, center, H, L, d, block, codes, scales, pooled, pooled_t, ldt, stream);
}

extern "C" int tb_kmean(const void *k, int dtype, int64_t H, int64_t L, int64_t d, float *kmean, void *stream) {
    TB_REQUIRE(dtype == TB_F32 || dtype == TB_BF16, "dtype must be f32 or bf16");
    if (H == 0 || d == 0) return TB_OK;
    TB_REQUIRE(L >= 1, "seq must be >= 1");
    cudaStream_t st = as_stream(stream);
    const size_t es = dtype == TB_F32 ? 4 : 2;
    const bool aligned = ((uintptr_t)k % 16 == 0) && ((L * d * es) % 16 == 0) && ((d * es) % 16 == 0);
    if (aligned && d == 128 && dtype == TB_BF16 && H * L < (1ll << 31)) {
        CUtensorMap tm;
        if (!make_tmap_2d(&tm, k, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 128, H * L, 256, 32, KM_CH,
                          CU_TENSOR_MAP_SWIZZLE_NONE))
            return fail(TB_ECUDA, "cuTensorMapEncodeTiled failed (kmean)");
        // 3 x 16 KB: the ring fits beside four kv_part CTAs per SM, so the chains start with the
        // step instead of waiting for kv_part's grid to drain (same-process graph A/B of the cfg4
        // step: 3 stages 0.15-0.2 ms faster than 6; TB_KM_STAGES overrides, tools only)
        int nst = 3;
        if (const char *e = getenv("TB_KM_STAGES")) nst = atoi(e) < 2 ? 2 : (atoi(e) > KM_STAGES ? KM_STAGES : atoi(e));
        const int smem = nst * KM_CH * 64;
        smem_attr(kmean_split_kernel, KM_STAGES * KM_CH * 64);
        kmean_split_kernel<<<dim3(4, (unsigned)H), 32, smem, st>>>(tm, L, nst, kmean);
    } else if (aligned && d <= 128) {
        constexpr int STAGES = 6;
        int chunk = (int)(16384 / (d * es));          // 16 KiB per stage
        if (chunk < 8) chunk = 8;
        size_t smem = (size_t)STAGES * chunk * d * es;
        if (dtype == TB_F32) {
            smem_attr(kmean_bulk_kernel<float, STAGES>, (int)smem);
            kmean_bulk_kernel<float, STAGES><<<(unsigned)H, 128, smem, st>>>((const float *)k, L, (int)d, chunk, kmean);
        } else {
            smem_attr(kmean_bulk_kernel<__nv_bfloat16, STAGES>, (int)smem);
            kmean_bulk_kernel<__nv_bfloat16, STAGES><<<(unsigned)H, 128, smem, st>>>((const __nv_bfloat16 *)k, L, (int)d, chunk, kmean);
        }
    } else {
        unsigned grid = (unsigned)cdiv(H * d, 128);
        if (dtype == TB_F32) kmean_simple_kernel<float><<<grid, 128, 0, st>>>((const float *)k, H, L, d, kmean);
        else kmean_simple_kernel<__nv_bfloat16><<<grid, 128, 0, st>>>((const __nv_bfloat16 *)k, H, L, d, kmean);
    }
    return check_launch("kmean");
}

extern "C" int tb_transpose_v(const void *v, int dtype, int64_t H, int64_t L, int64_t d, int64_t l_pad,
                              void *vt, void *stream) {
    TB_REQUIRE(l_pad >= L, "l_pad < L");
    if (H == 0 || d == 0 || l_pad == 0) return TB_OK;
    dim3 grid((unsigned)cdiv(l_pad, 32), (unsigned)cdiv(d, 32), (unsigned)H);
    cudaStream_t st = as_stream(stream);
    if (dtype == TB_F32) transpose_v_kernel<float><<<grid, dim3(32, 8), 0, st>>>((const float *)v, L, d, l_pad, (__nv_bfloat16 *)vt);
    else transpose_v_kernel<__nv_bfloat16><<<grid, dim3(32, 8), 0, st>>>((const __nv_bfloat16 *)v, L, d, l_pad, (__nv_bfloat16 *)vt);
    return check_launch("transpose_v");
}

extern "C" int tb_quantize_blockwise_planar(const void *x, int dtype, int64_t rows, int64_t cols, int8_t *q,
                                            float *scales, void *stream) {
    TB_REQUIRE(dtype == TB_F32 || dtype == TB_BF16, "dtype must be f32 or bf16");
    TB_REQUIRE(cols % 128 == 0 && ((uintptr_t)x % 16) == 0, "planar input needs cols % 128 == 0, 16-B aligned");
    if (rows == 0 || cols == 0) return TB_OK;
    const int64_t nbr = cdiv(rows, 128), nbc = cols / 128;
    TB_REQUIRE(nbr < 65536, "too many row blocks");
    dim3 grid((unsigned)nbc, (unsigned)nbr);
    cudaStream_t st = as_stream(stream);
    if (dtype == TB_F32)
        quantize_blockwise128_kernel<float, true><<<grid, 256, 0, st>>>((const float *)x, rows, cols, nbc, q, scales, nullptr);
    else
        quantize_blockwise128_kernel<__nv_bfloat16, true><<<grid, 256, 0, st>>>((const __nv_bfloat16 *)x, rows, cols, nbc, q,
                                                                                scales, nullptr);
    return check_launch("quantize_blockwise_planar");
}

// ---------------------------------------------------------------- FP8 V
// SURVEY.md §8 a17 (no reference function; the north star's "P/V to FP8"):
// V [H, L, d] -> e4m3 codes with one scale per head,
//   scale = f32(absmax(v[h])) / 448 (RN),  code = e4m3_rn_satfinite(v / safe)
// (safe = 1 for an all-zero head; IEEE divide).  Oracle:
// oracle/oracle.py quantize_v_fp8.  Two HBM passes: per-head absmax
// (uint-ordered atomicMax of non-negative floats), then the codes.
#include <cuda_fp8.h>
#include <algorithm>
namespace tb {
template <typename T>
__device__ __forceinline__ void vfp8_load8(const T *src, int64_t i, float (&x)[8]) {
    if constexpr (sizeof(T) == 2) {
        const uint4 w = __ldg(reinterpret_cast<const uint4 *>(src) + i);
        const __nv_bfloat162 *b = reinterpret_cast<const __nv_bfloat162 *>(&w);
#pragma unroll
        for (int u = 0; u < 4; u++) { const float2 f = __bfloat1622float2(b[u]); x[2 * u] = f.x; x[2 * u + 1] = f.y; }
    } else {
        const float4 a = __ldg(reinterpret_cast<const float4 *>(src) + 2 * i);
        const float4 b = __ldg(reinterpret_cast<const float4 *>(src) + 2 * i + 1);
        x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w; x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
    }
}

// Each CTA walks chunks of VB = 4 x 256 vectors (8 elements each): the four
// loads of a thread are issued before any use (4 x 16 B in flight per
// thread) and each load instruction is coalesced across the warp.
constexpr int VFP8_U = 4;
template <typename T>
__global__ void __launch_bounds__(256) vfp8_absmax_kernel(const T *__restrict__ v, int64_t per_head,
                                                          unsigned *__restrict__ am_bits) {
    const int h = blockIdx.y;
    const T *src = v + (int64_t)h * per_head;
    const int64_t nvec = per_head / 8;
    float am = 0.0f;
    for (int64_t c0 = (int64_t)blockIdx.x * 256 * VFP8_U; c0 < nvec; c0 += (int64_t)gridDim.x * 256 * VFP8_U) {
        float x[VFP8_U][8];
#pragma unroll
        for (int u = 0; u < VFP8_U; u++) {
            const int64_t i = c0 + u * 256 + threadIdx.x;
            if (i < nvec) vfp8_load8(src, i, x[u]);
            else {
#pragma unroll
                for (int e = 0; e < 8; e++) x[u][e] = 0.0f;
            }
        }
#pragma unroll
        for (int u = 0; u < VFP8_U; u++)
#pragma unroll
            for (int e = 0; e < 8; e++) am = fmaxf(am, fabsf(x[u][e]));
    }
    am = warp_max<32>(am);
    __shared__ float red[8];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = am;
    __syncthreads();
    if (threadIdx.x == 0) {
        float m = red[0];
        for (int w = 1; w < 8; w++) m = fmaxf(m, red[w]);
        atomicMax(am_bits + h, __float_as_uint(m));
    }
}

template <typename T>
__global__ void __launch_bounds__(256) vfp8_codes_kernel(const T *__restrict__ v, int64_t per_head,
                                                         const unsigned *__restrict__ am_bits,
                                                         uint8_t *__restrict__ codes, float *__restrict__ scales) {
    const int h = blockIdx.y;
    const float sc = __fdiv_rn(__uint_as_float(__ldg(am_bits + h)), 448.0f);
    if (blockIdx.x == 0 && threadIdx.x == 0) scales[h] = sc;
    const float safe = sc == 0.0f ? 1.0f : sc;
    const T *src = v + (int64_t)h * per_head;
    uint8_t *dst = codes + (int64_t)h * per_head;
    const int64_t nvec = per_head / 8;
    for (int64_t c0 = (int64_t)blockIdx.x * 256 * VFP8_U; c0 < nvec; c0 += (int64_t)gridDim.x * 256 * VFP8_U) {
        float x[VFP8_U][8];
#pragma unroll
        for (int u = 0; u < VFP8_U; u++) {
            const int64_t i = c0 + u * 256 + threadIdx.x;
            if (i < nvec) vfp8_load8(src, i, x[u]);
        }
#pragma unroll
        for (int u = 0; u < VFP8_U; u++) {
            const int64_t i = c0 + u * 256 + threadIdx.x;
            uint32_t w[2];
#pragma unroll
            for (int q = 0; q < 2; q++) {
                const __nv_fp8x2_storage_t lo = __nv_cvt_float2_to_fp8x2(
                    make_float2(__fdiv_rn(x[u][4 * q], safe), __fdiv_rn(x[u][4 * q + 1], safe)), __NV_SATFINITE, __NV_E4M3);
                const __nv_fp8x2_storage_t hi = __nv_cvt_float2_to_fp8x2(
                    make_float2(__fdiv_rn(x[u][4 * q + 2], safe), __fdiv_rn(x[u][4 * q + 3], safe)), __NV_SATFINITE,
                    __NV_E4M3);
                w[q] = (uint32_t)lo | ((uint32_t)hi << 16);
            }
            if (i < nvec) *reinterpret_cast<uint2 *>(dst + 8 * i) = make_uint2(w[0], w[1]);
        }
    }
}
}  // namespace tb

// am_ws: caller workspace of H uint32 (zeroed here on the stream)
extern "C" int tb_quant_v_fp8(const void *v, int dtype, int64_t H, int64_t L, int64_t d, uint8_t *codes,
                              float *scales, unsigned *am_ws, void *stream) {
    TB_REQUIRE(dtype == TB_F32 || dtype == TB_BF16, "dtype must be f32 or bf16");
    if (H == 0 || L == 0 || d == 0) return TB_OK;
    const int64_t per_head = L * d;
    TB_REQUIRE(per_head % 8 == 0, "seq * head_dim must be a multiple of 8");
    TB_REQUIRE((uintptr_t)v % 16 == 0 && (uintptr_t)codes % 8 == 0, "v must be 16-B and codes 8-B aligned");
    TB_REQUIRE(H <= 65535, "too many heads");
    cudaStream_t st = as_stream(stream);
    cudaMemsetAsync(am_ws, 0, H * sizeof(unsigned), st);
    const int64_t vecs = per_head / 8;
    // ~8 CTAs of 256 threads per SM in total over the heads
    unsigned gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(vecs, 256 * VFP8_U), cdiv(8 * 148, H)));
    dim3 grid(gx, (unsigned)H);
    if (dtype == TB_BF16) {
        vfp8_absmax_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>((const __nv_bfloat16 *)v, per_head, am_ws);
        vfp8_codes_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>((const __nv_bfloat16 *)v, per_head, am_ws, codes, scales);
    } else {
        vfp8_absmax_kernel<float><<<grid, 256, 0, st>>>((const float *)v, per_head, am_ws);
        vfp8_codes_kernel<float><<<grid, 256, 0, st>>>((const float *)v, per_head, am_ws, codes, scales);
    }
    return check_launch("quant_v_fp8");
}

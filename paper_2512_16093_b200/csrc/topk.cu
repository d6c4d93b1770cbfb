// topk.cu -- SLA block-importance: block scores + per-row top-k selection.
//
// Replaces select_topk_blocks (attention.py:269-284) and BlockMask.complement
// (attention.py:122-132).  Bit-exact contract:
//  * scores = qp . kp^T in OpenBLAS's order (oracle/tb_oracle.c
//    orc_block_scores): one fmaf chain from 0 over d for the regular sgemm
//    kernel; 16 lane chains + adjacent-pair tree for the small-matrix TN
//    kernel (nq*nkv <= 1200, d >= 32, nq*nkv*d <= 1e6).  CUDA cores, not
//    tensor cores: the order must match.
//  * selection = argsort(-s, stable)[:count]: the count largest, ties to the
//    lower index, -0.0 == +0.0; output ascending.  Radix select (4 x 8-bit
//    digits on order-preserving uint keys) per row, one warp per row.
#include "common.cuh"
#include "ptx.cuh"

#ifndef TB_TOPK_ROWS
#define TB_TOPK_ROWS 8
#endif
// kp loads in flight per thread (dims per batch) and CTAs per SM of the 8-row
// kernel: 4 x 16 B and three CTAs (64 registers) -- 0.334 vs 0.367 ms at cfg4
// for 8 and two CTAs (96 registers); 2 / 3 0.375, 4 / 4 and 2 / 4 spill
// (0.46-0.53) (tools/time_topk.py, interleaved A/B)
#ifndef TB_TOPK_KB
#define TB_TOPK_KB 4
#endif
#ifndef TB_TOPK_MINB
#define TB_TOPK_MINB 3
#endif

namespace tb {

__device__ __forceinline__ uint32_t desc_key(float s) {
    if (s == 0.0f) s = 0.0f;                          // canonicalise -0.0
    uint32_t u = __float_as_uint(s);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u); // larger float -> larger key
}

template <int R>
__global__ void __launch_bounds__(256) topk_kernel(
    const float *__restrict__ qp, const float *__restrict__ kp, int nq, int nkv, int d, int count,
    int small_path, int32_t *__restrict__ idx, uint8_t *__restrict__ comp, float *__restrict__ scores_out,
    __nv_bfloat16 *__restrict__ cov, int64_t cov_ld) {
    extern __shared__ __align__(16) uint8_t smem[];
    uint32_t *keys = reinterpret_cast<uint32_t *>(smem);                    // [R][nkv]
    float *qrow = reinterpret_cast<float *>(smem + (((size_t)R * nkv * 4 + 15) & ~(size_t)15));  // [R][d]
    const int h = blockIdx.y;
    const int row0 = blockIdx.x * R;
    const int nrows = min(R, nq - row0);
    for (int i = threadIdx.x; i < R * d; i += blockDim.x) {
        int r = i / d;
        qrow[i] = (r < nrows) ? qp[((int64_t)h * nq + row0 + r) * d + (i - r * d)] : 0.0f;
    }
    __syncthreads();
    const float *kph = kp + (int64_t)h * nkv * d;
    if (!small_path && (d & 3) == 0 && (((uintptr_t)kph) & 15) == 0) {
        // Regular-sgemm order (one fmaf chain per score over t ascending),
        // register-tiled: each thread owns JT kv columns x R rows and steps t
        // by 4 with float4 loads of kp and broadcast float4 reads of qp.
        constexpr int JT = 4;
        for (int j0 = threadIdx.x * JT; j0 < nkv; j0 += blockDim.x * JT) {
            float acc[R][JT];
#pragma unroll
            for (int r = 0; r < R; r++)
#pragma unroll
                for (int u = 0; u < JT; u++) acc[r][u] = 0.0f;
            const float *kr[JT];
#pragma unroll
            for (int u = 0; u < JT; u++) kr[u] = kph + (int64_t)min(j0 + u, nkv - 1) * d;
            for (int t = 0; t < d; t += 4) {
                float4 kv[JT];
#pragma unroll
                for (int u = 0; u < JT; u++) kv[u] = __ldg(reinterpret_cast<const float4 *>(kr[u] + t));
#pragma unroll
                for (int r = 0; r < R; r++) {
                    const float4 qv = *reinterpret_cast<const float4 *>(qrow + r * d + t);
#pragma unroll
                    for (int u = 0; u < JT; u++) {
                        acc[r][u] = __fmaf_rn(qv.x, kv[u].x, acc[r][u]);
                        acc[r][u] = __fmaf_rn(qv.y, kv[u].y, acc[r][u]);
                        acc[r][u] = __fmaf_rn(qv.z, kv[u].z, acc[r][u]);
                        acc[r][u] = __fmaf_rn(qv.w, kv[u].w, acc[r][u]);
                    }
                }
            }
#pragma unroll
            for (int r = 0; r < R; r++)
#pragma unroll
                for (int u = 0; u < JT; u++)
                    if (r < nrows && j0 + u < nkv) {
                        keys[r * nkv + j0 + u] = desc_key(acc[r][u]);
                        if (scores_out) scores_out[((int64_t)h * nq + row0 + r) * nkv + j0 + u] = acc[r][u];
                    }
        }
    } else
    for (int j = threadIdx.x; j < nkv; j += blockDim.x) {
        const float *kr = kph + (int64_t)j * d;
        float acc[R];
        if (!small_path) {
#pragma unroll
            for (int r = 0; r < R; r++) acc[r] = 0.0f;
            for (int t = 0; t < d; t++) {
                float kv = __ldg(kr + t);
#pragma unroll
                for (int r = 0; r < R; r++) acc[r] = __fmaf_rn(qrow[r * d + t], kv, acc[r]);
            }
        } else {
            for (int r = 0; r < R; r++) {
                float lane[16];
#pragma unroll
                for (int l = 0; l < 16; l++) lane[l] = 0.0f;
                for (int t = 0; t < d; t++) lane[t & 15] = __fmaf_rn(qrow[r * d + t], __ldg(kr + t), lane[t & 15]);
#pragma unroll
                for (int w = 8; w >= 1; w >>= 1)
#pragma unroll
                    for (int l = 0; l < w; l++) lane[l] = __fadd_rn(lane[2 * l], lane[2 * l + 1]);
                acc[r] = lane[0];
            }
        }
#pragma unroll
        for (int r = 0; r < R; r++) {
            if (r < nrows) {
                keys[r * nkv + j] = desc_key(acc[r]);
                if (scores_out) scores_out[((int64_t)h * nq + row0 + r) * nkv + j] = acc[r];
            }
        }
    }
    __syncthreads();

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int r = warp; r < nrows; r += 8) {
        const uint32_t *kr = keys + r * nkv;
        const int64_t row = (int64_t)h * nq + row0 + r;
        // Threshold key T = the count-th largest key: greedy bitwise search
        // from the MSB (32 rounds of a warp-wide count of keys >= candidate),
        // no atomics.  need = how many keys equal to T are taken.
        uint32_t T = 0;
        if (count < nkv) {
            for (int bit = 31; bit >= 0; bit--) {
                const uint32_t cand = T | (1u << bit);
                int c = 0;
                for (int j = lane; j < nkv; j += 32) c += kr[j] >= cand;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
                if (c >= count) T = cand;
            }
        }
        int need = count;
        if (count < nkv) {
            int gtc = 0;
            for (int j = lane; j < nkv; j += 32) gtc += kr[j] > T;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) gtc += __shfl_xor_sync(0xffffffffu, gtc, o);
            need = count - gtc;
        }
        // compaction in ascending index order
        const bool take_all = count >= nkv;
        int taken = 0, ties = 0;
        for (int base = 0; base < nkv; base += 32) {
            const int j = base + lane;
            const uint32_t k = (j < nkv) ? kr[j] : 0u;
            const bool valid = j < nkv;
            const bool gt = valid && (take_all || k > T);
            const bool eq = valid && !take_all && k == T;
            const unsigned eqb = __ballot_sync(0xffffffffu, eq);
            const int tie_rank = ties + __popc(eqb & ((1u << lane) - 1u));
            const bool sel = gt || (eq && tie_rank < need);
            const unsigned selb = __ballot_sync(0xffffffffu, sel);
            if (sel) idx[row * count + taken + __popc(selb & ((1u << lane) - 1u))] = j;
            if (comp && valid) comp[row * nkv + j] = sel ? 0 : 1;
            if (cov && valid) cov[row * cov_ld + j] = __float2bfloat16_rn(sel ? 0.0f : 1.0f);
            taken += __popc(selb);
            ties += __popc(eqb);
        }
        if (cov)
            for (int j = nkv + lane; j < cov_ld; j += 32) cov[row * cov_ld + j] = __float2bfloat16_rn(0.0f);
    }
}

// Fast path for the regular-sgemm order (d % 4 == 0, not the small-matrix
// kernel): 16 q rows per CTA, each thread JT kv columns x 16 rows with the
// chains packed in pairs of rows (fma.rn.f32x2 = two IEEE fmaf, bit-identical
// to the scalar chain), q staged transposed so a row pair is one 8-B load.
// Selection: 4-pass radix select (8-bit digits, warp-private histograms in
// shared memory) for the threshold key, then the same ballot compaction.
// Optional bf16 coverage output (1 = block in the complement) with row pitch
// cov_ld, zero-padded, the A operand of the linear branch's GEMM.
template <int JT, int R, int MINB>
__global__ void __launch_bounds__(320, MINB) topk16_kernel(
    const float *__restrict__ qp, const float *__restrict__ kpt, int64_t ldk, int nq, int nkv, int d, int count,
    int32_t *__restrict__ idx, uint8_t *__restrict__ comp, float *__restrict__ scores_out,
    __nv_bfloat16 *__restrict__ cov, int64_t cov_ld) {
    extern __shared__ __align__(16) uint8_t smem[];
    uint32_t *keys = reinterpret_cast<uint32_t *>(smem);                          // [R][nkv]
    float *qt = reinterpret_cast<float *>(smem + (((size_t)R * nkv * 4 + 15) & ~(size_t)15));   // [d][R]
    uint32_t *hist = reinterpret_cast<uint32_t *>(qt + (size_t)d * R);             // [warps][256]
    const int h = blockIdx.y;
    const int row0 = blockIdx.x * R;
    const int nrows = min(R, nq - row0);
    for (int i = threadIdx.x; i < R * d; i += blockDim.x) {
        const int r = i / d, t = i - r * d;
        qt[t * R + r] = (r < nrows) ? qp[((int64_t)h * nq + row0 + r) * d + t] : 0.0f;
    }
    __syncthreads();
    // kp transposed ([d][ldk] per head): a warp's float4 loads of 4 kv columns are contiguous
    const float *kth = kpt + (int64_t)h * d * ldk;
    for (int j0 = threadIdx.x * JT; j0 < nkv; j0 += blockDim.x * JT) {
        float2 acc[R / 2][JT];
#pragma unroll
        for (int r = 0; r < R / 2; r++)
#pragma unroll
            for (int u = 0; u < JT; u++) acc[r][u] = make_float2(0.0f, 0.0f);
        // TB_TOPK_KB dims per batch: the batch's coalesced float4 loads are all in flight before the FFMA2s
        auto step = [&](int t, const float4 kv) {
            const float4 *qrow = reinterpret_cast<const float4 *>(qt + t * R);
            float2 qpair[R / 2];
#pragma unroll
            for (int r4 = 0; r4 < R / 4; r4++) {
                const float4 q4 = qrow[r4];
                qpair[2 * r4] = make_float2(q4.x, q4.y);
                qpair[2 * r4 + 1] = make_float2(q4.z, q4.w);
            }
            const float kvu[4] = {kv.x, kv.y, kv.z, kv.w};
#pragma unroll
            for (int u = 0; u < JT; u++) {
                const float2 k2 = make_float2(kvu[u], kvu[u]);
#pragma unroll
                for (int r = 0; r < R / 2; r++) acc[r][u] = ptx::ffma2(qpair[r], k2, acc[r][u]);
            }
        };
        int t = 0;
        for (; t + TB_TOPK_KB <= d; t += TB_TOPK_KB) {
            float4 kv[TB_TOPK_KB];
#pragma unroll
            for (int i = 0; i < TB_TOPK_KB; i++) kv[i] = __ldg(reinterpret_cast<const float4 *>(kth + (int64_t)(t + i) * ldk + j0));
#pragma unroll
            for (int i = 0; i < TB_TOPK_KB; i++) step(t + i, kv[i]);
        }
        for (; t < d; t++) step(t, __ldg(reinterpret_cast<const float4 *>(kth + (int64_t)t * ldk + j0)));
#pragma unroll
        for (int r = 0; r < R / 2; r++)
#pragma unroll
            for (int u = 0; u < JT; u++) {
                const int j = j0 + u;
                if (j < nkv) {
                    if (2 * r < nrows) keys[(2 * r) * nkv + j] = desc_key(acc[r][u].x);
                    if (2 * r + 1 < nrows) keys[(2 * r + 1) * nkv + j] = desc_key(acc[r][u].y);
                    if (scores_out) {
                        if (2 * r < nrows) scores_out[((int64_t)h * nq + row0 + 2 * r) * nkv + j] = acc[r][u].x;
                        if (2 * r + 1 < nrows) scores_out[((int64_t)h * nq + row0 + 2 * r + 1) * nkv + j] = acc[r][u].y;
                    }
                }
            }
    }
    __syncthreads();

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t *hw = hist + warp * 256;
    const int nwarps = blockDim.x >> 5;
    for (int r = warp; r < nrows; r += nwarps) {
        const uint32_t *kr = keys + r * nkv;
        const int64_t row = (int64_t)h * nq + row0 + r;
        // threshold T = the count-th largest key, digit by digit from the top;
        // need = how many keys equal to T are taken
        uint32_t prefix = 0;
        int need = count;
        if (count < nkv) {
#pragma unroll 1
            for (int shift = 24; shift >= 0; shift -= 8) {
                for (int i = lane; i < 256; i += 32) hw[i] = 0;
                __syncwarp();
                const uint32_t hi_mask = shift == 24 ? 0u : (0xFFFFFFFFu << (shift + 8));
                for (int j = lane; j < nkv; j += 32) {
                    const uint32_t k = kr[j];
                    if ((k & hi_mask) == (prefix & hi_mask)) atomicAdd(&hw[(k >> shift) & 0xFF], 1u);
                }
                __syncwarp();
                // lane owns bins 255-8*lane .. 248-8*lane (descending); suffix counts from the top
                uint32_t c8[8], tot = 0;
#pragma unroll
                for (int i = 0; i < 8; i++) { c8[i] = hw[255 - 8 * lane - i]; tot += c8[i]; }
                uint32_t incl = tot;                       // inclusive scan over lanes (higher bins first)
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += v;
                }
                const uint32_t before = incl - tot;        // keys in bins above this lane's range
                // the bin where the running count first reaches need
                int hit = -1;
                uint32_t above = before;
                if (before < (uint32_t)need && incl >= (uint32_t)need) {
#pragma unroll
                    for (int i = 0; i < 8; i++) {
                        if (hit < 0) {
                            if (above + c8[i] >= (uint32_t)need) hit = i;
                            else above += c8[i];
                        }
                    }
                }
                const unsigned who = __ballot_sync(0xffffffffu, hit >= 0);
                const int src = __ffs(who) - 1;
                const int bin = __shfl_sync(0xffffffffu, 255 - 8 * lane - hit, src);
                const uint32_t ab = __shfl_sync(0xffffffffu, above, src);
                prefix |= (uint32_t)bin << shift;
                need -= (int)ab;
                __syncwarp();
            }
        }
        const uint32_t T = prefix;
        // compaction in ascending index order
        const bool take_all = count >= nkv;
        int taken = 0, ties = 0;
        for (int base = 0; base < nkv; base += 32) {
            const int j = base + lane;
            const uint32_t k = (j < nkv) ? kr[j] : 0u;
            const bool valid = j < nkv;
            const bool gt = valid && (take_all || k > T);
            const bool eq = valid && !take_all && k == T;
            const unsigned eqb = __ballot_sync(0xffffffffu, eq);
            const int tie_rank = ties + __popc(eqb & ((1u << lane) - 1u));
            const bool sel = gt || (eq && tie_rank < need);
            const unsigned selb = __ballot_sync(0xffffffffu, sel);
            if (sel) idx[row * count + taken + __popc(selb & ((1u << lane) - 1u))] = j;
            if (comp && valid) comp[row * nkv + j] = sel ? 0 : 1;
            if (cov && valid) cov[row * cov_ld + j] = __float2bfloat16_rn(sel ? 0.0f : 1.0f);
            taken += __popc(selb);
            ties += __popc(eqb);
        }
        if (cov)
            for (int j = nkv + lane; j < cov_ld; j += 32) cov[row * cov_ld + j] = __float2bfloat16_rn(0.0f);
    }
}

}  // namespace tb

using namespace tb;

static int topk_launch(const float *qp, const float *kp, const float *kpt, int64_t ldk, int64_t H, int64_t nq,
                       int64_t nkv, int64_t d, int64_t count, int32_t *idx, uint8_t *comp, float *scores_out,
                       __nv_bfloat16 *cov, int64_t cov_ld, cudaStream_t st) {
    TB_REQUIRE(count >= 1 && count <= nkv, "count must be in [1, num_kv_blocks]");
    TB_REQUIRE(nkv <= 16384, "num_kv_blocks > 16384 unsupported");
    TB_REQUIRE(d >= 1 && d <= 1024, "head_dim out of range");
    if (H == 0 || nq == 0) return TB_OK;
    const double mnk = (double)nq * (double)nkv * (double)d;
    const int small = (nq * nkv <= 1200 && d >= 32 && mnk <= 1e6) ? 1 : 0;
    const bool fast16 = !small && kpt != nullptr && ldk % 4 == 0 && ldk >= cdiv(nkv, 4) * 4 &&
                        (((uintptr_t)kpt) % 16) == 0 && nkv <= 2560;
    if (fast16) {
        constexpr int JT = 4;                        // 320 threads x 4 columns >= 1182 kv blocks (cfg4) in one pass
        constexpr int R = TB_TOPK_ROWS;              // q rows per CTA (8: TB_TOPK_MINB CTAs per SM)
        const size_t smem = (((size_t)R * nkv * 4 + 15) & ~(size_t)15) + (size_t)d * R * 4 + 10 * 256 * 4;
        dim3 grid((unsigned)cdiv(nq, R), (unsigned)H);
        smem_attr(topk16_kernel<JT, R, R == 16 ? 1 : (R == 8 ? TB_TOPK_MINB : 3)>, (int)smem);
        topk16_kernel<JT, R, R == 16 ? 1 : (R == 8 ? TB_TOPK_MINB : 3)><<<grid, 320, smem, st>>>(qp, kpt, ldk, (int)nq, (int)nkv, (int)d, (int)count, idx, comp,
                                                  scores_out, cov, cov_ld);
        return check_launch("topk16");
    }
#define TB_TOPK(R)                                                                                 \
    {                                                                                              \
        size_t smem = (((size_t)(R) * nkv * 4 + 15) & ~(size_t)15) + (size_t)(R) * d * 4;          \
        smem_attr(topk_kernel<R>, (int)smem); \
        dim3 grid((unsigned)cdiv(nq, R), (unsigned)H);                                             \
        topk_kernel<R><<<grid, 256, smem, st>>>(qp, kp, (int)nq, (int)nkv, (int)d, (int)count, small, \
                                                idx, comp, scores_out, cov, cov_ld);               \
    }
    if (nkv <= 2048) TB_TOPK(8) else if (nkv <= 4096) TB_TOPK(4) else TB_TOPK(1)
#undef TB_TOPK
    return check_launch("topk_blocks");
}

extern "C" int tb_topk_blocks(const float *qp, const float *kp, int64_t H, int64_t nq, int64_t nkv, int64_t d,
                              int64_t count, int32_t *idx, uint8_t *comp, float *scores_out, void *stream) {
    return topk_launch(qp, kp, nullptr, 0, H, nq, nkv, d, count, idx, comp, scores_out, nullptr, 0, as_stream(stream));
}

extern "C" int tb_topk_blocks_cov(const float *qp, const float *kp, const float *kpt, int64_t ldk, int64_t H,
                                  int64_t nq, int64_t nkv, int64_t d, int64_t count, int32_t *idx, uint8_t *comp,
                                  void *cov, int64_t cov_ld, void *stream) {
    TB_REQUIRE(cov != nullptr && cov_ld >= nkv && cov_ld % 8 == 0, "cov needs a row pitch >= nkv, multiple of 8");
    return topk_launch(qp, kp, kpt, ldk, H, nq, nkv, d, count, idx, comp, nullptr, (__nv_bfloat16 *)cov, cov_ld,
                       as_stream(stream));
}

// ---------------------------------------------------------------------------
// Pair union of the top-k lists (q_block 64 on the tensor-core attention
// kernel, which runs 128-row tiles = two 64-row q-blocks).  For tile t the
// ascending lists of q-blocks 2t and 2t+1 (attention.py:269-284 indices) are
// merged into one ascending list of distinct kv blocks; entry = block |
// (mask << 28), mask bit 0 = selected by q-block 2t, bit 1 = by 2t+1.  The
// kernel visits each union block once and zeroes P for the rows whose q-block
// did not select it, so every row still attends exactly its own top-k set.
// One warp per (head, tile): merge-with-duplicates positions by binary
// search (pos(a_i) = i + #{b < a_i}, pos(b_j) = j + #{a <= b_j}: equal values
// land adjacent, A first), then a ballot compaction that folds each equal
// pair into one entry with both bits.
namespace tb {
__global__ void __launch_bounds__(32) pair_union_kernel(const int32_t *__restrict__ idx, int nq, int count,
                                                        int32_t *__restrict__ out, int32_t *__restrict__ cnt,
                                                        int ld) {
    extern __shared__ int32_t mrg[];             // 2 * count merged entries: (value << 2) | source bit
    const int lane = threadIdx.x;
    const int t = blockIdx.x, h = blockIdx.y, ntile = gridDim.x;
    const int32_t *A = idx + ((int64_t)h * nq + 2 * t) * count;
    const bool hasB = 2 * t + 1 < nq;
    const int32_t *B = A + count;
    const int nb = hasB ? count : 0;
    for (int i = lane; i < count; i += 32) {
        const int32_t a = A[i];
        int lo = 0, hi = nb;                      // #{b < a}
        while (lo < hi) { const int m = (lo + hi) >> 1; if (B[m] < a) lo = m + 1; else hi = m; }
        mrg[i + lo] = (a << 2) | 1;
    }
    for (int j = lane; j < nb; j += 32) {
        const int32_t b = B[j];
        int lo = 0, hi = count;                   // #{a <= b}
        while (lo < hi) { const int m = (lo + hi) >> 1; if (A[m] <= b) lo = m + 1; else hi = m; }
        mrg[j + lo] = (b << 2) | 2;
    }
    __syncwarp();
    const int n = count + nb;
    int32_t *o = out + ((int64_t)h * ntile + t) * ld;
    int taken = 0;
    for (int base = 0; base < n; base += 32) {
        const int m = base + lane;
        int32_t e = 0;
        bool keep = false;
        if (m < n) {
            e = mrg[m];
            keep = m == 0 || (mrg[m - 1] >> 2) != (e >> 2);
            if (keep && m + 1 < n && (mrg[m + 1] >> 2) == (e >> 2)) e |= mrg[m + 1] & 3;
        }
        const unsigned kb = __ballot_sync(0xffffffffu, keep);
        if (keep) o[taken + __popc(kb & ((1u << lane) - 1u))] = (e >> 2) | ((e & 3) << 28);
        taken += __popc(kb);
    }
    if (lane == 0) cnt[(int64_t)h * ntile + t] = taken;
}
}  // namespace tb

extern "C" int tb_pair_union(const int32_t *idx, int64_t H, int64_t nq, int64_t count, int32_t *pair_idx,
                             int32_t *pair_cnt, int64_t pair_ld, void *stream) {
    TB_REQUIRE(count >= 1 && pair_ld >= 2 * count, "pair_ld must be >= 2 * count");
    TB_REQUIRE(count <= 4096, "count > 4096 unsupported");
    if (H == 0 || nq == 0) return TB_OK;
    dim3 grid((unsigned)cdiv(nq, 2), (unsigned)H);
    const size_t smem = (size_t)2 * count * 4;
    smem_attr(pair_union_kernel, (int)smem);
    pair_union_kernel<<<grid, 32, smem, as_stream(stream)>>>(idx, (int)nq, (int)count, pair_idx, pair_cnt,
                                                              (int)pair_ld);
    return check_launch("pair_union");
}

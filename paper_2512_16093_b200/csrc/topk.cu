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

namespace tb {

__device__ __forceinline__ uint32_t desc_key(float s) {
    if (s == 0.0f) s = 0.0f;                          // canonicalise -0.0
    uint32_t u = __float_as_uint(s);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u); // larger float -> larger key
}

template <int R>
__global__ void __launch_bounds__(256) topk_kernel(
    const float *__restrict__ qp, const float *__restrict__ kp, int nq, int nkv, int d, int count,
    int small_path, int32_t *__restrict__ idx, uint8_t *__restrict__ comp, float *__restrict__ scores_out) {
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
            taken += __popc(selb);
            ties += __popc(eqb);
        }
    }
}

}  // namespace tb

using namespace tb;

extern "C" int tb_topk_blocks(const float *qp, const float *kp, int64_t H, int64_t nq, int64_t nkv, int64_t d,
                              int64_t count, int32_t *idx, uint8_t *comp, float *scores_out, void *stream) {
    TB_REQUIRE(count >= 1 && count <= nkv, "count must be in [1, num_kv_blocks]");
    TB_REQUIRE(nkv <= 16384, "num_kv_blocks > 16384 unsupported");
    TB_REQUIRE(d >= 1 && d <= 1024, "head_dim out of range");
    if (H == 0 || nq == 0) return TB_OK;
    const double mnk = (double)nq * (double)nkv * (double)d;
    const int small = (nq * nkv <= 1200 && d >= 32 && mnk <= 1e6) ? 1 : 0;
    cudaStream_t st = as_stream(stream);
#define TB_TOPK(R)                                                                                 \
    {                                                                                              \
        size_t smem = (((size_t)(R) * nkv * 4 + 15) & ~(size_t)15) + (size_t)(R) * d * 4;          \
        cudaFuncSetAttribute(topk_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
        dim3 grid((unsigned)cdiv(nq, R), (unsigned)H);                                             \
        topk_kernel<R><<<grid, 256, smem, st>>>(qp, kp, (int)nq, (int)nkv, (int)d, (int)count, small, \
                                                idx, comp, scores_out);                            \
    }
    if (nkv <= 2048) TB_TOPK(8) else if (nkv <= 4096) TB_TOPK(4) else TB_TOPK(1)
#undef TB_TOPK
    return check_launch("topk_blocks");
}

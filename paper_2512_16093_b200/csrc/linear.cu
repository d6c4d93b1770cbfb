// linear.cu -- the SLA linear branch's per-block operand on tcgen05 (sm_100a).
//
// kv_part[h, b] = [V_b | 1]^T phi(K_b)  for every kv block b of every head
// (attention.py:320-325: phi(K_b)^T V_b and the denominator sum phi(K_b)),
// stored bf16 [H, nkv, dx, d] with rows 0..d-1 = V_b^T phi(K_b) (v channel x
// k channel), row d = sum_t phi(K_b)[t, :], rows d+1..dx-1 zero -- the B
// operand of the coverage GEMM kv_sel = cov . kv_part (attention.py:326-328).
//
// One CTA per (kv block, head), 128 threads, up to four CTAs per SM:
//   * TMA loads the K and V tiles (64 tokens x 128 channels bf16, two
//     64-channel 128B-swizzled boxes each; tokens >= L arrive as zeros)
//   * the threads apply phi in place on the K tile (elementwise, so the
//     swizzle does not matter; padded tokens -> 0, not phi(0)) and sum the
//     denominator row in f32
//   * one thread issues 4 x tcgen05.mma kind::f16 M128 N128 K16 with both
//     operands MN-major (channel-contiguous): D[v][k] = sum_t V[t][v] phi(K)[t][k]
//   * the f32 accumulator goes TMEM -> registers -> bf16 swizzled smem tile
//     -> TMA store (two 64-column boxes)
// The kernel is HBM-bound: 32 KB read + (dx*d*2) B written per block.
// Optionally (tb_linear_kv_part_pool) it also emits the raw K block means
// (pool_block_means) and their transposed copy from the tile it already holds,
// which saves the separate K pooling pass over HBM on the top-k's path.
#include "common.cuh"
#include "ptx.cuh"
#include "tmap.cuh"

namespace tb {

namespace lkv {
constexpr int BN = 64, D = 128, THREADS = 128;
constexpr uint32_t TILE = BN * D * 2;        // 16 KB (bf16)
struct Smem {
    uint8_t k[TILE];                         // phi(K) tile, later the output tile (first half)
    uint8_t v[TILE];                         // V tile, later the output tile (second half)
    uint64_t full, mma_done;
    uint32_t tmem_base;
    float red[4];                            // per warp: absmax of the centered K values (K codes)
};
constexpr size_t SMEM_BYTES = sizeof(Smem);
}  // namespace lkv

__device__ __forceinline__ float phi_f(float x) { return x >= 0.0f ? x + 1.0f : __expf(x); }

__global__ void __launch_bounds__(lkv::THREADS) kv_part_kernel(const __grid_constant__ CUtensorMap tm_k,
                                                                const __grid_constant__ CUtensorMap tm_v,
                                                                const __grid_constant__ CUtensorMap tm_out,
                                                                int L, int nkv, int dx,
                                                                __nv_bfloat16 *__restrict__ kv_part,
                                                                float *__restrict__ kp, float *__restrict__ kpt,
                                                                int64_t ldt, const float *__restrict__ km,
                                                                int8_t *__restrict__ kc, float *__restrict__ ks) {
    using namespace lkv;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    Smem &S = *reinterpret_cast<Smem *>(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int b = blockIdx.x, h = blockIdx.y;
    const int64_t row0 = ((int64_t)h * nkv + b) * dx;          // first output row of this block
    if (threadIdx.x == 0) {
        if (ptx::smem_u32(smem_raw) & 1023) __trap();
        ptx::mbar_init(&S.full, 1);
        ptx::mbar_init(&S.mma_done, 1);
        ptx::fence_barrier_init();
        ptx::mbar_arrive_expect_tx(&S.full, 2 * TILE);
        ptx::tma_load_3d(S.k, &tm_k, 0, b * BN, h, &S.full);
        ptx::tma_load_3d(S.k + TILE / 2, &tm_k, 64, b * BN, h, &S.full);
        ptx::tma_load_3d(S.v, &tm_v, 0, b * BN, h, &S.full);
        ptx::tma_load_3d(S.v + TILE / 2, &tm_v, 64, b * BN, h, &S.full);
    }
    if (warp == 0) ptx::tmem_alloc<128>(&S.tmem_base);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = S.tmem_base;

    // rows d+1 .. dx-1 of the block are zero (padding of the GEMM's N)
    for (int i = threadIdx.x; i < (dx - D - 1) * (D / 8); i += THREADS) {
        const int r = D + 1 + i / (D / 8), c = (i % (D / 8)) * 8;
        *reinterpret_cast<uint4 *>(kv_part + (row0 + r) * D + c) = make_uint4(0u, 0u, 0u, 0u);
    }
    ptx::mbar_wait(&S.full, 0);
    if (kp != nullptr) {
        // the raw K block's mean per channel (pool_block_means, attention.py:256-266) from
        // the tile already in shared memory, in numpy's reduceat order: seed + 8-accumulator
        // pairwise body + sequential tail (as pool_quant_tile_kernel); thread = channel
        const int c = threadIdx.x, e = min(BN, L - b * BN);
        const uint8_t *colp = S.k + (c >> 6) * (TILE / 2) + (c & 7) * 2;
        const int g = (c & 63) >> 3;
        // K codes (optional): absmax of the k_mean-centered values, order-free, on the same reads
        const float ctr = kc ? __ldg(km + h * D + c) : 0.0f;
        float am = 0.0f;
        auto ld = [&](int t) {
            const float x = __bfloat162float(*reinterpret_cast<const __nv_bfloat16 *>(colp + t * 128 + ((g ^ (t & 7)) * 16)));
            am = fmaxf(am, fabsf(__fsub_rn(x, ctr)));
            return x;
        };
        const float seed = ld(0);
        const int n = e - 1;
        float res = -0.0f;
        if (n >= 8) {
            float r[8];
#pragma unroll
            for (int j = 0; j < 8; j++) r[j] = ld(1 + j);
            const int full8 = n - (n % 8);
            for (int i = 8; i < full8; i += 8) {
#pragma unroll
                for (int j = 0; j < 8; j++) r[j] = __fadd_rn(r[j], ld(1 + i + j));
            }
            res = __fadd_rn(__fadd_rn(__fadd_rn(r[0], r[1]), __fadd_rn(r[2], r[3])),
                            __fadd_rn(__fadd_rn(r[4], r[5]), __fadd_rn(r[6], r[7])));
            for (int i = full8; i < n; i++) res = __fadd_rn(res, ld(1 + i));
        } else {
            for (int i = 0; i < n; i++) res = __fadd_rn(res, ld(1 + i));
        }
        const float pm = __fdiv_rn(n > 0 ? __fadd_rn(seed, res) : seed, (float)e);
        kp[((int64_t)h * nkv + b) * D + c] = pm;
        if (kpt) kpt[((int64_t)h * D + c) * ldt + b] = pm;   // [H][d][ldt]: the top-k kernel's coalesced operand
        if (kc) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) am = fmaxf(am, __shfl_xor_sync(0xffffffffu, am, o));
            if (lane == 0) S.red[warp] = am;
        }
        __syncthreads();                                   // every read of the raw tile before phi overwrites it
    }
    // the K block's scale (quantize_token_blocks, attention.py:201-220), as pool_quant_tile_kernel
    float qsafe = 1.0f, qinv = 1.0f;
    bool qexact = false;
    float qctr[8];
    if (kc) {
        const float s = quant_scale(fmaxf(fmaxf(S.red[0], S.red[1]), fmaxf(S.red[2], S.red[3])));
        if (threadIdx.x == 0) ks[(int64_t)h * nkv + b] = s;
        qsafe = (s == 0.0f) ? 1.0f : s;
        qinv = __frcp_rn(qsafe);
        qexact = !(qsafe >= 1.17549435e-38f && qinv <= 3.0e38f);   // subnormal scale: exact division
        const int c0 = (threadIdx.x >> 6) * 64 + ((threadIdx.x >> 3) & 7) * 8;
#pragma unroll
        for (int i = 0; i < 8; i++) qctr[i] = __ldg(km + h * D + c0 + i);
    }
    {
        // phi in place: thread = (channel half, 8-channel group g, 8-token slice tq)
        const int half = threadIdx.x >> 6, g = (threadIdx.x >> 3) & 7, tq = threadIdx.x & 7;
        float den[8];
#pragma unroll
        for (int i = 0; i < 8; i++) den[i] = 0.0f;
#pragma unroll
        for (int tt = 0; tt < 8; tt++) {
            const int t = tq * 8 + tt;
            uint4 *p = reinterpret_cast<uint4 *>(S.k + half * (TILE / 2) + t * 128 + ((g ^ (t & 7)) * 16));
            uint4 w = *p;
            __nv_bfloat162 *bw = reinterpret_cast<__nv_bfloat162 *>(&w);
            const bool in = b * BN + t < L;
            if (kc && in) {                               // codes of the raw (centered) values before phi
                float xv[8];
#pragma unroll
                for (int i = 0; i < 4; i++) {
                    const float2 x = __bfloat1622float2(bw[i]);
                    xv[2 * i] = __fsub_rn(x.x, qctr[2 * i]);
                    xv[2 * i + 1] = __fsub_rn(x.y, qctr[2 * i + 1]);
                }
                uint32_t cw[2];
                quant_fast_n<8>(xv, qsafe, qinv, qexact, cw);
                *reinterpret_cast<uint2 *>(kc + ((int64_t)h * L + b * BN + t) * D + half * 64 + g * 8) =
                    make_uint2(cw[0], cw[1]);
            }
#pragma unroll
            for (int i = 0; i < 4; i++) {
                const float2 x = __bfloat1622float2(bw[i]);
                const float f0 = in ? phi_f(x.x) : 0.0f, f1 = in ? phi_f(x.y) : 0.0f;
                den[2 * i] += f0;
                den[2 * i + 1] += f1;
                bw[i] = __floats2bfloat162_rn(f0, f1);
            }
            *p = w;
        }
#pragma unroll
        for (int i = 0; i < 8; i++) {
            den[i] += __shfl_xor_sync(0xffffffffu, den[i], 1);
            den[i] += __shfl_xor_sync(0xffffffffu, den[i], 2);
            den[i] += __shfl_xor_sync(0xffffffffu, den[i], 4);
        }
        if (tq == 0) {
            uint4 w;
            __nv_bfloat162 *bw = reinterpret_cast<__nv_bfloat162 *>(&w);
#pragma unroll
            for (int i = 0; i < 4; i++) bw[i] = __floats2bfloat162_rn(den[2 * i], den[2 * i + 1]);
            *reinterpret_cast<uint4 *>(kv_part + (row0 + D) * D + half * 64 + g * 8) = w;
        }
    }
    ptx::fence_async_smem();                 // phi(K) (generic writes) -> tensor-core reads
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == 0) {
        if (ptx::elect_one()) {
            // A = V tile (M = v channel, MN-major), B = phi(K) tile (N = k channel, MN-major), K = tokens
            constexpr uint32_t ID = ptx::idesc_bf16(128, D) | (1u << 15) | (1u << 16);
            const uint64_t ad = ptx::sdesc_sw128_mn(ptx::smem_u32(S.v), TILE / 2, 1024);
            const uint64_t bd = ptx::sdesc_sw128_mn(ptx::smem_u32(S.k), TILE / 2, 1024);
#pragma unroll
            for (int k = 0; k < BN / 16; k++) ptx::mma_f16(tmem, ad + 128 * k, bd + 128 * k, ID, k > 0 ? 1u : 0u);
            ptx::mma_commit(&S.mma_done);
        }
        __syncwarp();
    }
    ptx::mbar_wait(&S.mma_done, 0);
    ptx::tc_fence_after();
    // accumulator row r = v channel (TMEM lane) -> bf16 -> 128B-swizzled [128 x 64] boxes in smem
    {
        const int r = warp * 32 + lane;
        const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16);
#pragma unroll 1
        for (int c = 0; c < D; c += 32) {
            uint32_t x0[16], x1[16];
            ptx::tmem_ld16(taddr + c, x0);
            ptx::tmem_ld16(taddr + c + 16, x1);
            ptx::tmem_wait_ld();
            uint32_t w[16];
#pragma unroll
            for (int i = 0; i < 8; i++) {
                __nv_bfloat162 p0 = __floats2bfloat162_rn(__uint_as_float(x0[2 * i]), __uint_as_float(x0[2 * i + 1]));
                __nv_bfloat162 p1 = __floats2bfloat162_rn(__uint_as_float(x1[2 * i]), __uint_as_float(x1[2 * i + 1]));
                w[i] = *reinterpret_cast<uint32_t *>(&p0);
                w[8 + i] = *reinterpret_cast<uint32_t *>(&p1);
            }
            // columns c..c+31 = four 16-byte chunks u of box (c / 64)
            uint8_t *box = (c < 64 ? S.k : S.v);
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const int u = ((c & 63) >> 3) + q;
                *reinterpret_cast<uint4 *>(box + r * 128 + ((u ^ (r & 7)) * 16)) =
                    make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
            }
        }
    }
    ptx::fence_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) {
        ptx::tma_store_2d(&tm_out, S.k, 0, (int)row0);
        ptx::tma_store_2d(&tm_out, S.v, 64, (int)row0);
        ptx::bulk_commit();
        ptx::bulk_wait_read0();
    }
    if (warp == 0) ptx::tmem_dealloc<128>(tmem);
}

}  // namespace tb

using namespace tb;

extern "C" int tb_linear_kv_part_codes(const void *k, const void *v, int64_t H, int64_t L, int64_t d,
                                       int64_t kv_block, int64_t dx, void *kv_part, float *kp, float *kpt,
                                       int64_t ldt, const float *k_mean, int8_t *k_codes, float *k_scales,
                                       void *stream) {
    using namespace lkv;
    TB_REQUIRE((k_codes == nullptr) == (k_scales == nullptr) && (k_codes == nullptr || k_mean != nullptr),
               "k_codes, k_scales and k_mean go together");
    TB_REQUIRE(k_codes == nullptr || kp != nullptr, "K codes come with the K pool (kp)");
    TB_REQUIRE(k_codes == nullptr || ((uintptr_t)k_codes % 8) == 0, "unaligned k_codes");
    TB_REQUIRE(kpt == nullptr || (kp != nullptr && ldt >= cdiv(L, kv_block)), "kpt needs kp and ldt >= blocks");
    TB_REQUIRE(d == D && kv_block == BN, "tb_linear_kv_part: d == 128 and kv_block == 64 only");
    TB_REQUIRE(dx > d && dx * d % 256 == 0, "dx must exceed d with dx*d a multiple of 256");
    TB_REQUIRE(((uintptr_t)k % 16) == 0 && ((uintptr_t)v % 16) == 0 && ((uintptr_t)kv_part % 16) == 0, "unaligned");
    if (H == 0 || L == 0) return TB_OK;
    const int64_t nkv = cdiv(L, BN);
    TB_REQUIRE(H * nkv * dx < (1ll << 31), "too many rows for a 2-D tensor map");
    CUtensorMap tk, tv, to;
    if (!make_tmap_3d(&tk, k, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, D, L, H, D * 2, L * D * 2, 64, BN, 1) ||
        !make_tmap_3d(&tv, v, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, D, L, H, D * 2, L * D * 2, 64, BN, 1) ||
        !make_tmap_2d(&to, kv_part, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, D, H * nkv * dx, D * 2, 64, 128))
        return fail(TB_ECUDA, "cuTensorMapEncodeTiled failed (kv_part)");
    cudaStream_t st = as_stream(stream);
    smem_attr(kv_part_kernel, (int)SMEM_BYTES);
    kv_part_kernel<<<dim3((unsigned)nkv, (unsigned)H), THREADS, SMEM_BYTES, st>>>(
        tk, tv, to, (int)L, (int)nkv, (int)dx, (__nv_bfloat16 *)kv_part, kp, kpt, ldt, k_mean, k_codes, k_scales);
    return check_launch("kv_part");
}

extern "C" int tb_linear_kv_part_pool(const void *k, const void *v, int64_t H, int64_t L, int64_t d,
                                      int64_t kv_block, int64_t dx, void *kv_part, float *kp, float *kpt,
                                      int64_t ldt, void *stream) {
    return tb_linear_kv_part_codes(k, v, H, L, d, kv_block, dx, kv_part, kp, kpt, ldt, nullptr, nullptr, nullptr,
                                   stream);
}

extern "C" int tb_linear_kv_part(const void *k, const void *v, int64_t H, int64_t L, int64_t d, int64_t kv_block,
                                 int64_t dx, void *kv_part, void *stream) {
    return tb_linear_kv_part_pool(k, v, H, L, d, kv_block, dx, kv_part, nullptr, nullptr, 0, stream);
}

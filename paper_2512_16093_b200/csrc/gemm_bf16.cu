// gemm_bf16.cu -- batched bf16 GEMM on tcgen05 for the SLA linear branch
// (a 1-SM kernel, and the transposed CTA-pair kernel below that serves the
// coverage GEMM's shape: bf16 output, N % 256 == 0).
//
// C[h] (M x N) = A[h] (M x K, K-major) . B[h] (K x N, N-contiguous = MN-major)
// with f32 accumulation in TMEM.  Used for kv_sel = cov . kv_part
// (attention.py:326-328): A = the complement mask (0/1, exact in bf16),
// B = the per-kv-block phi(K_b)^T [V_b|1] matrices; M = #q-blocks,
// K = #kv-blocks, N = (d+16)*d.  Replaces a cuBLAS batched GEMM.
//
// Persistent CTAs (one per SM), warp-specialised like the W8A8 kernel:
// warp 0 TMA producer (A tile 128x64 K-major SW128; B tile 64x256 as four
// 64-column MN-major SW128 atoms), warp 1 single-thread MMA issuer
// (4 x kind::f16 M128 N256 K16 per 64-deep stage), 8 epilogue warps draining
// a double-buffered 2 x 256-column f32 TMEM accumulator to bf16/f32.
#include <cstdlib>

#include "common.cuh"
#include "ptx.cuh"
#include "tmap.cuh"

namespace tb {

namespace gbf {
constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4;
constexpr int EPI_WARPS = 8;
constexpr int THREADS = 64 + EPI_WARPS * 32;
constexpr uint32_t A_BYTES = BM * BK * 2;   // 16 KiB
constexpr uint32_t B_BYTES = BK * BN * 2;   // 32 KiB
struct Smem {
    uint8_t a[STAGES][A_BYTES];
    uint8_t b[STAGES][B_BYTES];
    uint64_t full[STAGES], empty[STAGES];
    uint64_t acc_full[2], acc_empty[2];
    uint32_t tmem_base;
};
constexpr size_t SMEM_BYTES = sizeof(Smem) + 1024;
}  // namespace gbf

template <bool OUT_F32>
__global__ void __launch_bounds__(gbf::THREADS, 1) gemm_bf16_kernel(
    const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b, void *__restrict__ C,
    int H, int M, int N, int K, int64_t ldc, int64_t c_batch) {
    using namespace gbf;
    extern __shared__ uint8_t smem_raw[];
    Smem &S = *reinterpret_cast<Smem *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nmt = (M + BM - 1) / BM, nnt = N / BN, nkb = (K + BK - 1) / BK;
    const int tiles_per_head = nmt * nnt;
    const int ntiles = H * tiles_per_head;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < STAGES; s++) { ptx::mbar_init(&S.full[s], 1); ptx::mbar_init(&S.empty[s], 1); }
        for (int b = 0; b < 2; b++) { ptx::mbar_init(&S.acc_full[b], 1); ptx::mbar_init(&S.acc_empty[b], EPI_WARPS * 32); }
        ptx::fence_barrier_init();
        ptx::prefetch_tmap(&tma_a);
        ptx::prefetch_tmap(&tma_b);
    }
    if (warp == 1) ptx::tmem_alloc<512>(&S.tmem_base);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = S.tmem_base;

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                const int h = tile / tiles_per_head, rem = tile % tiles_per_head;
                const int nt = rem / nmt, mt = rem % nmt;       // m fastest: B tile reused from L2
                for (int kb = 0; kb < nkb; kb++) {
                    ptx::mbar_wait_sleep(&S.empty[stage], phase ^ 1);
                    ptx::mbar_arrive_expect_tx(&S.full[stage], A_BYTES + B_BYTES);
                    ptx::tma_load_3d(S.a[stage], &tma_a, kb * BK, mt * BM, h, &S.full[stage]);
#pragma unroll
                    for (int q = 0; q < BN / 64; q++)
                        ptx::tma_load_3d(S.b[stage] + q * (BK * 128), &tma_b, nt * BN + q * 64, kb * BK, h,
                                         &S.full[stage]);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            int stage = 0, buf = 0;
            uint32_t phase = 0, bphase = 0;
            constexpr uint32_t idesc = ptx::idesc_bf16(BM, BN) | (1u << 16);   // B MN-major
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                ptx::mbar_wait_sleep(&S.acc_empty[buf], bphase ^ 1);
                ptx::tc_fence_after();
                for (int kb = 0; kb < nkb; kb++) {
                    ptx::mbar_wait_sleep(&S.full[stage], phase);
                    ptx::tc_fence_after();
                    const uint64_t ad = ptx::sdesc_sw128(ptx::smem_u32(S.a[stage]));
                    const uint64_t bd = ptx::sdesc_sw128_mn(ptx::smem_u32(S.b[stage]), BK * 128, 1024);
#pragma unroll
                    for (int k = 0; k < BK / 16; k++)   // K=16: A +32 B in the row, B +16 rows (2048 B)
                        ptx::mma_f16(tmem + buf * BN, ad + 2 * k, bd + 128 * k, idesc, (kb > 0 || k > 0) ? 1u : 0u);
                    ptx::mma_commit(&S.empty[stage]);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
                ptx::mma_commit(&S.acc_full[buf]);
                buf ^= 1;
                if (buf == 0) bphase ^= 1;
            }
        }
    } else {
        const int ew = warp - 2;
        const int quarter = warp & 3;
        const int half = ew >> 2;                 // 128-column half of the 256-wide tile
        const int trow = quarter * 32 + lane;
        int buf = 0;
        uint32_t bphase = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            const int h = tile / tiles_per_head, rem = tile % tiles_per_head;
            const int nt = rem / nmt, mt = rem % nmt;
            ptx::mbar_wait_sleep(&S.acc_full[buf], bphase);
            ptx::tc_fence_after();
            const int row = mt * BM + trow;
            const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + buf * BN + half * 128;
#pragma unroll 1
            for (int c = 0; c < 128; c += 32) {
                uint32_t r0[16], r1[16];
                ptx::tmem_ld16(taddr + c, r0);
                ptx::tmem_ld16(taddr + c + 16, r1);
                ptx::tmem_wait_ld();
                if (row < M) {
                    const int64_t off = (int64_t)h * c_batch + (int64_t)row * ldc + nt * BN + half * 128 + c;
                    if constexpr (OUT_F32) {
                        float *o = reinterpret_cast<float *>(C) + off;
#pragma unroll
                        for (int i = 0; i < 16; i += 4) {
                            *reinterpret_cast<float4 *>(o + i) = make_float4(__uint_as_float(r0[i]), __uint_as_float(r0[i + 1]),
                                                                             __uint_as_float(r0[i + 2]), __uint_as_float(r0[i + 3]));
                            *reinterpret_cast<float4 *>(o + 16 + i) = make_float4(__uint_as_float(r1[i]), __uint_as_float(r1[i + 1]),
                                                                                  __uint_as_float(r1[i + 2]), __uint_as_float(r1[i + 3]));
                        }
                    } else {
                        __nv_bfloat16 *o = reinterpret_cast<__nv_bfloat16 *>(C) + off;
                        uint32_t w[16];
#pragma unroll
                        for (int i = 0; i < 8; i++) {
                            __nv_bfloat162 a = __floats2bfloat162_rn(__uint_as_float(r0[2 * i]), __uint_as_float(r0[2 * i + 1]));
                            __nv_bfloat162 b = __floats2bfloat162_rn(__uint_as_float(r1[2 * i]), __uint_as_float(r1[2 * i + 1]));
                            w[i] = *reinterpret_cast<uint32_t *>(&a);
                            w[8 + i] = *reinterpret_cast<uint32_t *>(&b);
                        }
#pragma unroll
                        for (int i = 0; i < 16; i += 4)
                            *reinterpret_cast<uint4 *>(o + 2 * i) = make_uint4(w[i], w[i + 1], w[i + 2], w[i + 3]);
                    }
                }
            }
            ptx::tc_fence_before();
            ptx::mbar_arrive(&S.acc_empty[buf]);
            buf ^= 1;
            if (buf == 0) bphase ^= 1;
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) ptx::tmem_dealloc<512>(tmem);
}

// ---------------------------------------------------------------------------
// Transposed CTA-pair kernel for the coverage GEMM's shape (few rows M = nq,
// very wide N = (d+2)*d, K = nkv): computes C^T = B^T . A^T, so the wide
// dimension becomes the pair's M = 256 (128 rows per SM, N % 256 == 0: no
// padding) and the short one the MMA's N (split into near-equal tiles of <= 256
// columns rounded to 16: 591 -> 208 + 208 + 176).  Per SM and 64-deep stage the
// TMA brings 16 KB of B^T (MN-major: B is N-contiguous) and half of the A^T
// tile (K-major), and each half of A^T is read once for both SMs of the pair:
// ~60 KB of shared-memory traffic per 4 MMAs instead of the 1-SM kernel's 96 KB
// per 4 MMAs of the same size, which is what bounded it (tensor pipe 64%).
// The epilogue writes C row q, columns e..e+31 per warp and TMEM column: each
// thread holds one e (its TMEM lane), 16 q columns per tcgen05.ld.
namespace gbt {
constexpr int BMH = 128, BK = 64, STAGES = 6, EPI_WARPS = 8;
constexpr int THREADS = 64 + EPI_WARPS * 32;
constexpr int BH_MAX = 128;                                  // B^T rows per SM (N tile / 2)
struct Smem {
    uint8_t a[STAGES][BMH * BK * 2];                         // 2 MN-major 64-wide chunks of 8 KB
    uint8_t b[STAGES][BH_MAX * BK * 2];                      // K-major rows of A (= columns of C^T)
    uint64_t full[STAGES], empty[STAGES];
    uint64_t acc_full[2], acc_empty[2];
    uint32_t tmem_base;
};
constexpr size_t SMEM_BYTES = sizeof(Smem) + 1024;
static_assert(SMEM_BYTES <= 232448, "transposed GEMM shared memory over 227 KB");
}  // namespace gbt

__device__ __forceinline__ void gbt_tile(int tile, int nmt, int nnt, int &h, int &mt, int &nt) {
    const int per = nmt * nnt;
    h = tile / per;
    const int r = tile - h * per;
    nt = r / nmt;
    mt = r - nt * nmt;                                       // wide-dimension tile fastest: the A^T tile is reused from L2
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(gbt::THREADS, 1) gemm_bf16_t2_kernel(
    const __grid_constant__ CUtensorMap tma_bt, const __grid_constant__ CUtensorMap tma_at, __nv_bfloat16 *__restrict__ C,
    int H, int M, int N, int K, int ntf, int bh, int64_t ldc, int64_t c_batch) {
    using namespace gbt;
    extern __shared__ uint8_t smem_raw[];
    Smem &S = *reinterpret_cast<Smem *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = ptx::cluster_ctarank();
    const int cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
    const int nmt = N / (2 * BMH), nnt = (M + ntf - 1) / ntf, nkb = (K + BK - 1) / BK;
    const int ntiles = H * nmt * nnt;
    const uint32_t stage_tx = 2u * (uint32_t)(BMH * BK * 2 + bh * BK * 2);   // both CTAs' boxes

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < STAGES; s++) { ptx::mbar_init(&S.full[s], 1); ptx::mbar_init(&S.empty[s], 1); }
        for (int b = 0; b < 2; b++) { ptx::mbar_init(&S.acc_full[b], 1); ptx::mbar_init(&S.acc_empty[b], 2 * EPI_WARPS); }
        ptx::fence_barrier_init();
        ptx::prefetch_tmap(&tma_bt);
        ptx::prefetch_tmap(&tma_at);
    }
    if (warp == 1) ptx::tmem_alloc_pair<512>(&S.tmem_base);
    ptx::tc_fence_before();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    const uint32_t tmem = S.tmem_base;

    if (warp == 0) {
        if (ptx::elect_one()) {
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = cluster; tile < ntiles; tile += nclusters) {
                int h, mt, nt;
                gbt_tile(tile, nmt, nnt, h, mt, nt);
                const int q0 = nt * ntf, nw = min(ntf, ((M - q0 + 15) / 16) * 16);
                const int e0 = mt * 2 * BMH + (int)rank * BMH;
                for (int kb = 0; kb < nkb; kb++) {
                    ptx::mbar_wait_sleep(&S.empty[stage], phase ^ 1);
                    const uint32_t fullc = ptx::mapa(ptx::smem_u32(&S.full[stage]), 0);
                    if (rank == 0) ptx::mbar_arrive_expect_tx(&S.full[stage], stage_tx);
                    ptx::tma_load_3d_pair(S.a[stage], &tma_bt, e0, kb * BK, h, fullc);
                    ptx::tma_load_3d_pair(S.a[stage] + BK * 128, &tma_bt, e0 + 64, kb * BK, h, fullc);
                    ptx::tma_load_3d_pair(S.b[stage], &tma_at, kb * BK, q0 + (int)rank * (nw / 2), h, fullc);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (rank == 0) {
            int stage = 0, buf = 0;
            uint32_t phase = 0, bphase = 0;
            for (int tile = cluster; tile < ntiles; tile += nclusters) {
                int h, mt, nt;
                gbt_tile(tile, nmt, nnt, h, mt, nt);
                const int q0 = nt * ntf, nw = min(ntf, ((M - q0 + 15) / 16) * 16);
                const uint32_t idesc = ptx::idesc_bf16(2 * BMH, nw) | (1u << 15);   // A (= B^T) MN-major
                ptx::mbar_wait_sleep(&S.acc_empty[buf], bphase);
                ptx::tc_fence_after();
                for (int kb = 0; kb < nkb; kb++) {
                    ptx::mbar_wait_sleep(&S.full[stage], phase);
                    ptx::tc_fence_after();
                    const uint64_t ad = ptx::sdesc_sw128_mn(ptx::smem_u32(S.a[stage]), BK * 128, 1024);
                    const uint64_t bd = ptx::sdesc_sw128(ptx::smem_u32(S.b[stage]));
                    if (ptx::elect_one()) {
#pragma unroll
                        for (int k = 0; k < BK / 16; k++)   // K16: A +16 rows (2 KB), B +32 B in the row
                            ptx::mma_f16_pair(tmem + buf * 256, ad + 128 * k, bd + 2 * k, idesc, (kb > 0 || k > 0) ? 1u : 0u);
                        ptx::mma_commit_pair(&S.empty[stage], 0x3);
                        if (kb == nkb - 1) ptx::mma_commit_pair(&S.acc_full[buf], 0x3);
                    }
                    __syncwarp();
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
                buf ^= 1;
                if (buf == 0) bphase ^= 1;
            }
        }
    } else {
        const int wu = __shfl_sync(0xffffffffu, warp, 0);
        const int ew = wu - 2, quarter = wu & 3, half = ew >> 2;
        const uint32_t acc_empty0 = ptx::mapa(ptx::smem_u32(&S.acc_empty[0]), 0);
        const uint32_t acc_empty1 = ptx::mapa(ptx::smem_u32(&S.acc_empty[1]), 0);
        int buf = 0;
        uint32_t bphase = 0;
#pragma unroll
        for (int b = 0; b < 2; b++) {                        // both accumulators start free
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive_cluster(b ? acc_empty1 : acc_empty0);
        }
        for (int tile = cluster; tile < ntiles; tile += nclusters) {
            int h, mt, nt;
            gbt_tile(tile, nmt, nnt, h, mt, nt);
            const int q0 = nt * ntf, nw = min(ntf, ((M - q0 + 15) / 16) * 16);
            const int ng = nw / 16, g0 = half ? (ng + 1) / 2 : 0, g1 = half ? ng : (ng + 1) / 2;
            const int e = mt * 2 * BMH + (int)rank * BMH + quarter * 32 + lane;
            __nv_bfloat16 *cp = C + (int64_t)h * c_batch + (int64_t)q0 * ldc + e;
            ptx::mbar_wait_sleep(&S.acc_full[buf], bphase);
            ptx::tc_fence_after();
            const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + buf * 256;
#pragma unroll 1
            for (int g = g0; g < g1; g++) {
                uint32_t r[16];
                ptx::tmem_ld16(taddr + g * 16, r);
                ptx::tmem_wait_ld();
                const int qn = min(16, M - q0 - g * 16);
#pragma unroll
                for (int i = 0; i < 16; i++)
                    if (i < qn) cp[(int64_t)(g * 16 + i) * ldc] = __float2bfloat16_rn(__uint_as_float(r[i]));
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive_cluster(buf ? acc_empty1 : acc_empty0);
            buf ^= 1;
            if (buf == 0) bphase ^= 1;
        }
    }
    ptx::tc_fence_before();
    ptx::cluster_sync();
    if (warp == 1) ptx::tmem_dealloc_pair<512>(tmem);
}

int num_sms();

}  // namespace tb

using namespace tb;

extern "C" int tb_gemm_bf16_batched(const void *A, const void *B, void *C, int64_t H, int64_t M, int64_t N, int64_t K,
                                    int64_t lda, int64_t ldb, int64_t ldc, int out_dtype, void *stream) {
    using namespace gbf;
    TB_REQUIRE(N % BN == 0, "N must be a multiple of 256");
    TB_REQUIRE(lda % 8 == 0 && ldb % 8 == 0 && ldc % 8 == 0, "leading dims must be multiples of 8");
    TB_REQUIRE(lda >= K && ldb >= N && ldc >= N, "leading dims too small");
    TB_REQUIRE(((uintptr_t)A % 16) == 0 && ((uintptr_t)B % 16) == 0 && ((uintptr_t)C % 16) == 0, "unaligned");
    if (H == 0 || M == 0) return TB_OK;
    // TB_GEMM_T2=0 keeps the 1-SM kernel (A/B)
    static const bool use_t2 = [] { const char *e = getenv("TB_GEMM_T2"); return !e || atoi(e) != 0; }();
    if (use_t2 && out_dtype == TB_BF16 && N % 256 == 0 && K >= 1 && (ldc * 2) % 16 == 0) {
        // transposed CTA-pair kernel: B^T [H][N][K] read MN-major from B, A read K-major
        const int64_t nnt = cdiv(M, 256);
        // near-equal column tiles, multiples of 16 (591 -> 208 + 208 + 176: 0.655 ms at cfg4, vs
        // 0.686 for 256 + 256 + 80 and 0.667-0.749 for 224 / 192 / 160-wide tiles)
        const int64_t ntf = cdiv(cdiv(M, nnt), 16) * 16;
        const int bh = (int)(ntf / 2 < 8 ? 8 : (ntf / 2 + 7) / 8 * 8);
        CUtensorMap tbt, tat;
        if (!make_tmap_3d(&tbt, B, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, N, K, H, ldb * 2, ldb * 2 * K, 64, gbt::BK, 1) ||
            !make_tmap_3d(&tat, A, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, K, M, H, lda * 2, lda * 2 * M, gbt::BK, bh, 1))
            return fail(TB_ECUDA, "cuTensorMapEncodeTiled failed (gemm_bf16_t2)");
        const int64_t ntiles = H * (N / 256) * cdiv(M, ntf);
        const int64_t pairs = num_sms() / 2;
        const int grid = 2 * (int)(ntiles < pairs ? ntiles : pairs);
        smem_attr(gemm_bf16_t2_kernel, (int)gbt::SMEM_BYTES);
        gemm_bf16_t2_kernel<<<grid, gbt::THREADS, gbt::SMEM_BYTES, as_stream(stream)>>>(
            tbt, tat, reinterpret_cast<__nv_bfloat16 *>(C), (int)H, (int)M, (int)N, (int)K, (int)ntf, bh, ldc, ldc * M);
        return check_launch("gemm_bf16_t2");
    }
    CUtensorMap ta, tbm;
    // A [H][M][K] (row pitch lda), B [H][K][N] (row pitch ldb), both bf16
    if (!make_tmap_3d(&ta, A, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, K, M, H, lda * 2, lda * 2 * M, BK, BM, 1) ||
        !make_tmap_3d(&tbm, B, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, N, K, H, ldb * 2, ldb * 2 * K, 64, BK, 1))
        return fail(TB_ECUDA, "cuTensorMapEncodeTiled failed (gemm_bf16)");
    const int64_t ntiles = H * cdiv(M, BM) * (N / BN);
    const int grid = (int)(ntiles < num_sms() ? ntiles : num_sms());
    cudaStream_t st = as_stream(stream);
    if (out_dtype == TB_F32) {
        smem_attr(gemm_bf16_kernel<true>, (int)SMEM_BYTES);
        gemm_bf16_kernel<true><<<grid, THREADS, SMEM_BYTES, st>>>(ta, tbm, C, (int)H, (int)M, (int)N, (int)K, ldc, ldc * M);
    } else {
        smem_attr(gemm_bf16_kernel<false>, (int)SMEM_BYTES);
        gemm_bf16_kernel<false><<<grid, THREADS, SMEM_BYTES, st>>>(ta, tbm, C, (int)H, (int)M, (int)N, (int)K, ldc, ldc * M);
    }
    return check_launch("gemm_bf16");
}

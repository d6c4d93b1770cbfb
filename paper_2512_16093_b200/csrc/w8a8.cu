// w8a8.cu -- W8A8 INT8 GEMM with 128x128 block scales.
//
// Replaces w8a8_matmul (blockquant.py:132-161) and the GEMM of
// quantized_linear_forward (blockquant.py:164-182):
//   out[i,j] = sum_{kb ascending} (f32(seg_kb[i,j]) * sa[i/128,kb]) * sb[kb,j/128]
//   (+ bias[j]),  seg_kb = exact integer code dot over k-block kb.
//
// tcgen05 path (block 128, K%128==0, N%128==0): persistent CTAs, one per SM,
// warp-specialised: warp 0 issues TMA loads of 128x128 A / B^T code tiles
// (128B swizzle) into a 4-stage ring; warp 1 issues 4 x tcgen05.mma
// kind::i8 (M=128,N=128,K=32) per k-block into one of two s32 TMEM segment
// buffers; 8 epilogue warps drain each segment (tcgen05.ld), promote it
// into f32 register accumulators with the per-block scales, and store.
// Exact mode reproduces the reference rounding sequence bit-for-bit (seg ->
// f32 exactly via the 1.5*2^23 magic, then two RN multiplies and an RN add);
// fast mode folds the two scales into one FMA (tolerance-level).
#include <cstdlib>

#include <cstring>

#include "common.cuh"
#include "ptx.cuh"
#include "tmap.cuh"

// exact promotion: (seg * sa) * sb with the second product as a packed FMA with
// a +0 addend (A/B knob; 0 = two scalar multiplies)
#ifndef TB_W8_EXACT_FMA0
#define TB_W8_EXACT_FMA0 1
#endif

namespace tb {

// ------------------------------------------------------------ tcgen05 path
namespace gemm {
#ifndef TB_W8_EPI_WARPS
#define TB_W8_EPI_WARPS 8
#endif
constexpr int EPI_WARPS = TB_W8_EPI_WARPS;       // 8 or 16 (column groups of BN / (EPI_WARPS / 4))
constexpr int BM = 128, BK = 128, STAGES = EPI_WARPS == 16 ? 3 : 4;
constexpr int THREADS = 64 + EPI_WARPS * 32;
template <int BN>
struct Smem {
    uint8_t a[STAGES][BM * BK];
    uint8_t b[STAGES][BN * BK];
    uint64_t full[STAGES], empty[STAGES];
    uint64_t seg_full[2], seg_empty[2];
    uint32_t tmem_base;
    alignas(1024) uint8_t stage_out[EPI_WARPS][32 * 128];   // per-warp 32 rows x 128 B output chunk (SW128)
};
template <int BN>
constexpr size_t smem_bytes() { return sizeof(Smem<BN>) + 1024; }
}  // namespace gemm

// BN = 128 or 256 (tile 128 x BN, s32 segment buffers 2 x BN TMEM columns).
// Each epilogue warp owns 32 rows (its TMEM lane quarter) x BN/2 columns;
// a BN/2 column span never crosses a 128-column scale block.
// plane > 0: the output is stored as N/plane planes [M, plane] (plane | 128):
// a qkv projection lands head-major ([3, H, M, head_dim]) for the attention
// with no permute.  act == 1: GELU (tanh form, sampler.py:55-58) on the result.
__device__ __forceinline__ float gelu_tanh(float x) {
    float t;
    const float u = 0.7978845608028654f * fmaf(0.044715f * x, x * x, x);
    asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(u));
    return 0.5f * x * (1.0f + t);
}

template <int BN, bool EXACT, bool OUT_BF16>
__global__ void __launch_bounds__(gemm::THREADS, 1) w8a8_tc_kernel(
    const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
    const __grid_constant__ CUtensorMap tma_out,
    const float *__restrict__ sa, const float *__restrict__ sb, const float *__restrict__ bias,
    void *__restrict__ out, int M, int N, int K, int plane, int act) {
    using namespace gemm;
    constexpr int CW = BN / (EPI_WARPS / 4);
    constexpr uint32_t TMEM_COLS = 2 * BN;
    extern __shared__ uint8_t smem_raw[];
    Smem<BN> &S = *reinterpret_cast<Smem<BN> *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nmt = (M + BM - 1) / BM, nnt = N / BN, nkb = K / BK, nnb = N / 128;
    const int ntiles = nmt * nnt;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < STAGES; s++) { ptx::mbar_init(&S.full[s], 1); ptx::mbar_init(&S.empty[s], 1); }
        for (int b = 0; b < 2; b++) { ptx::mbar_init(&S.seg_full[b], 1); ptx::mbar_init(&S.seg_empty[b], EPI_WARPS * 32); }
        ptx::fence_barrier_init();
        ptx::prefetch_tmap(&tma_a);
        ptx::prefetch_tmap(&tma_b);
    }
    if (warp == 1) ptx::tmem_alloc<TMEM_COLS>(&S.tmem_base);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = S.tmem_base;

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                const int mt = tile / nnt, nt = tile % nnt;   // n fastest: A band reused from L2, B (weights) L2-resident
                for (int kb = 0; kb < nkb; kb++) {
                    ptx::mbar_wait_sleep(&S.empty[stage], phase ^ 1);
                    ptx::mbar_arrive_expect_tx(&S.full[stage], (BM + BN) * BK);
                    ptx::tma_load_2d(S.a[stage], &tma_a, kb * BK, mt * BM, &S.full[stage]);
                    ptx::tma_load_2d(S.b[stage], &tma_b, kb * BK, nt * BN, &S.full[stage]);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            int stage = 0, buf = 0;
            uint32_t phase = 0, bphase = 0;
            constexpr uint32_t idesc = ptx::idesc_i8(BM, BN);
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                for (int kb = 0; kb < nkb; kb++) {
                    ptx::mbar_wait_sleep(&S.seg_empty[buf], bphase ^ 1);
                    ptx::mbar_wait_sleep(&S.full[stage], phase);
                    ptx::tc_fence_after();
                    const uint64_t ad = ptx::sdesc_sw128(ptx::smem_u32(S.a[stage]));
                    const uint64_t bd = ptx::sdesc_sw128(ptx::smem_u32(S.b[stage]));
#pragma unroll
                    for (int k = 0; k < BK / 32; k++)   // K=32 bytes per kind::i8 MMA -> +2 in desc units
                        ptx::mma_i8(tmem + buf * BN, ad + 2 * k, bd + 2 * k, idesc, k > 0 ? 1u : 0u);
                    ptx::mma_commit(&S.empty[stage]);
                    ptx::mma_commit(&S.seg_full[buf]);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                    buf ^= 1;
                    if (buf == 0) bphase ^= 1;
                }
            }
        }
    } else {
        const int ew = warp - 2;
        const int quarter = warp & 3;          // TMEM lanes this warp may touch
        const int half = ew >> 2;              // column group of the tile
        const int trow = quarter * 32 + lane;
        int buf = 0;
        uint32_t bphase = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            const int mt = tile / nnt, nt = tile % nnt;   // n fastest: A band reused from L2, B (weights) L2-resident
            const int col0 = nt * BN + half * CW;
            const int nb = col0 / 128;
            float2 acc2[CW / 2];
#pragma unroll
            for (int i = 0; i < CW / 2; i++) acc2[i] = make_float2(0.0f, 0.0f);
            float s_a = __ldg(sa + (size_t)mt * nkb), s_b = __ldg(sb + nb);
            for (int kb = 0; kb < nkb; kb++) {
                const float2 sa2 = make_float2(s_a, s_a), sb2 = make_float2(s_b, s_b);
                const float2 sab2 = make_float2(s_a * s_b, s_a * s_b);
                if (kb + 1 < nkb) {                     // prefetch next k-block's scales
                    s_a = __ldg(sa + (size_t)mt * nkb + kb + 1);
                    s_b = __ldg(sb + (size_t)(kb + 1) * nnb + nb);
                }
                ptx::mbar_wait_sleep(&S.seg_full[buf], bphase);
                ptx::tc_fence_after();
                const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + buf * BN + half * CW;
                // 16-column chunks, double-buffered: the tcgen05.ld of chunk c+1 is in
                // flight while chunk c is promoted (wait::ld covers all outstanding loads)
#ifdef TB_W8_NOEPI
                ptx::tc_fence_before();
                ptx::mbar_arrive(&S.seg_empty[buf]);
                buf ^= 1;
                if (buf == 0) bphase ^= 1;
                continue;
#endif
                uint32_t rb[2][16];
                ptx::tmem_ld16(taddr, rb[0]);
                ptx::tmem_wait_ld();
#pragma unroll
                for (int c = 0; c < CW / 16; c++) {
                    if (c + 1 < CW / 16) ptx::tmem_ld16(taddr + (c + 1) * 16, rb[(c + 1) & 1]);
                    const uint32_t (&r)[16] = rb[c & 1];
#pragma unroll
                    for (int i = 0; i < 16; i += 2) {
                        // exact s32 -> f32 (|seg| <= 128*127^2 < 2^22).  Fast mode splits the
                        // conversion between pipes: 3 of 4 pairs by I2FP (ALU), 1 of 4 by the
                        // 1.5*2^23 magic + FADD2 (FMA pipe)
                        float2 x;
                        if (!EXACT && (i & 6) == 6) {
                            const float2 m = make_float2(__int_as_float((int)r[i] + 0x4B400000),
                                                         __int_as_float((int)r[i + 1] + 0x4B400000));
                            x = ptx::fadd2(m, make_float2(-12582912.0f, -12582912.0f));
                        } else {
                            x = make_float2(__int2float_rn((int)r[i]), __int2float_rn((int)r[i + 1]));
                        }
                        float2 &o = acc2[(c * 16 + i) >> 1];
                        if constexpr (EXACT) {
                            // the reference sequence bit-for-bit: packed RN ops round each
                            // lane like the scalar op, but ptxas contracts a packed multiply
                            // feeding a packed add into FFMA2 (tools/ubench_f32x2.cu), so the
                            // product that feeds the add is formed with scalar RN multiplies
                            const float2 p = ptx::fmul2(x, sa2);
#if TB_W8_EXACT_FMA0
                            // p * sb as a packed FMA with a +0 addend: the RN product except
                            // that -0 becomes +0, which cannot change o (it starts at +0, and
                            // x + (+0) == x + (-0) for every x != -0); ptxas neither folds it
                            // into a multiply nor contracts it into the add
                            o = ptx::fadd2(o, ptx::ffma2(p, sb2, make_float2(0.0f, 0.0f)));
#else
                            o = ptx::fadd2(o, make_float2(__fmul_rn(p.x, sb2.x), __fmul_rn(p.y, sb2.y)));
#endif
                        } else {
                            o = ptx::ffma2(x, sab2, o);
                        }
                    }
                    ptx::tmem_wait_ld();
                }
                ptx::tc_fence_before();
                ptx::mbar_arrive(&S.seg_empty[buf]);             // segment buffer free for the MMA
                buf ^= 1;
                if (buf == 0) bphase ^= 1;
            }
            if (bias) {
#pragma unroll
                for (int i = 0; i < CW / 2; i++) {
                    acc2[i].x = __fadd_rn(acc2[i].x, __ldg(bias + col0 + 2 * i));
                    acc2[i].y = __fadd_rn(acc2[i].y, __ldg(bias + col0 + 2 * i + 1));
                }
            }
            // stores: each warp stages 32 rows x 128 B (32 f32 or 64 bf16 columns) in a
            // 128B-swizzled smem chunk and one lane TMA-stores it (rows >= M are clipped)
            if (act == 1) {
#pragma unroll
                for (int i = 0; i < CW / 2; i++) { acc2[i].x = gelu_tanh(acc2[i].x); acc2[i].y = gelu_tanh(acc2[i].y); }
            }
            constexpr int CPC = OUT_BF16 ? 64 : 32;             // columns per chunk
            uint8_t *stg = S.stage_out[ew];
            const uint32_t stg_s = ptx::smem_u32(stg);
            const int row0 = mt * BM + quarter * 32;
#pragma unroll
            for (int ch = 0; ch < CW / CPC; ch++) {
                if (lane == 0) ptx::bulk_wait_read0();          // previous chunk has left the buffer
                __syncwarp();
#pragma unroll
                for (int u = 0; u < 8; u++) {                   // 8 x 16-byte units per 128-B row
                    uint32_t w0, w1, w2, w3;
                    if constexpr (OUT_BF16) {
                        const int p = (ch * CPC + 8 * u) >> 1;     // first float2 of the unit
                        __nv_bfloat162 b0 = __floats2bfloat162_rn(acc2[p].x, acc2[p].y);
                        __nv_bfloat162 b1 = __floats2bfloat162_rn(acc2[p + 1].x, acc2[p + 1].y);
                        __nv_bfloat162 b2 = __floats2bfloat162_rn(acc2[p + 2].x, acc2[p + 2].y);
                        __nv_bfloat162 b3 = __floats2bfloat162_rn(acc2[p + 3].x, acc2[p + 3].y);
                        w0 = *reinterpret_cast<uint32_t *>(&b0); w1 = *reinterpret_cast<uint32_t *>(&b1);
                        w2 = *reinterpret_cast<uint32_t *>(&b2); w3 = *reinterpret_cast<uint32_t *>(&b3);
                    } else {
                        const int p = (ch * CPC + 4 * u) >> 1;
                        w0 = __float_as_uint(acc2[p].x); w1 = __float_as_uint(acc2[p].y);
                        w2 = __float_as_uint(acc2[p + 1].x); w3 = __float_as_uint(acc2[p + 1].y);
                    }
                    const uint32_t dst = stg_s + lane * 128 + ((u ^ (lane & 7)) * 16);
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" :: "r"(dst), "r"(w0), "r"(w1), "r"(w2),
                                 "r"(w3) : "memory");
                }
                ptx::fence_async_smem();
                __syncwarp();
                if (lane == 0) {
                    const int c = col0 + ch * CPC;
                    if (plane) ptx::tma_store_3d(&tma_out, stg, c % plane, row0, c / plane);
                    else ptx::tma_store_2d(&tma_out, stg, c, row0);
                    ptx::bulk_commit();
                }
            }
        }
        if (lane == 0) ptx::bulk_wait_read0();
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) ptx::tmem_dealloc<TMEM_COLS>(tmem);
}

// ------------------------------------------------------- 2-SM tcgen05 path
// CTA pairs (cluster 2x1): each pair computes a 256 x 256 output tile with
// tcgen05.mma.cta_group::2 (M = 256, each CTA supplies 128 rows of A and 128
// of the 256 B rows, each CTA's TMEM receives its 128 rows x 256 columns).
// Per SM and k-block that is 16 KB of A + 16 KB of B through shared memory
// instead of 16 + 32 KB: the single-SM kernel is bound by that operand traffic
// (TB_W8_NOEPI: ~2 POPS without any epilogue).  The leader CTA (rank 0) owns
// the operand-full and segment-free barriers and issues the MMAs; commits are
// multicast to both CTAs; both CTAs' epilogues drain their own TMEM rows with
// the same promotion as the single-SM kernel and TMA-store their rows.
// Epilogue width: EPW = 8 (two warps per SM sub-partition, 128 columns each)
// or 16 (four per sub-partition, 64 columns each).  The promotion is
// latency-bound at ~200 instructions per warp per k-block (ncu source view:
// fixed-latency and TMEM-load dependencies, profiles/r02_source_level_stalls.md),
// so 16 warps hide twice the latency; the register file then allows 112 per
// epilogue thread (64 accumulators + a 16-column TMEM group).  The quantizing
// epilogue (OUTM 2) keeps EPW = 8 (its 128x128 block absmax spans one warp
// quarter-set).  Fast mode converts every s32 segment with I2FP: re-seeding
// TMEM with 1.5*2^23 for FADD2 conversions (or IMAD-based ones) measured
// 1.5-7% slower in same-box A/B runs.
namespace gemm2 {
constexpr int BM = 128, BN = 256, BK = 128;
template <int EPW>
struct Cfg {
    static constexpr int THREADS = 128 + EPW * 32;
    // warpgroup 0: TMA warp, MMA warp, two idle warps; the rest: epilogue.
    // setmaxnreg moves the control warpgroup's registers to the epilogue
    // (each role's code sits inside the branch that resized it)
    // setmaxnreg only moves registers inside the CTA's launch allocation
    // (THREADS x LAUNCH_REGS): what the control warpgroup releases must cover
    // what the epilogue warps acquire, or the increase waits forever
    static constexpr int LAUNCH_REGS = (65536 / THREADS) / 8 * 8;
    static constexpr int CTRL_REGS = EPW == 8 ? 56 : 32;
    static constexpr int EPI_REGS = EPW == 8 ? 224 : 112;
    static constexpr int STAGES = EPW == 8 ? 5 : 4;
    static constexpr bool STG2 = EPW == 8;                      // second staging buffer per warp
    static constexpr int CW = BN / (EPW / 4);                    // columns per epilogue warp
};
static_assert(128 * (Cfg<8>::LAUNCH_REGS - Cfg<8>::CTRL_REGS) >= 32 * 8 * (Cfg<8>::EPI_REGS - Cfg<8>::LAUNCH_REGS) &&
                  128 * (Cfg<16>::LAUNCH_REGS - Cfg<16>::CTRL_REGS) >=
                      32 * 16 * (Cfg<16>::EPI_REGS - Cfg<16>::LAUNCH_REGS),
              "setmaxnreg budget: the control warps must release what the epilogue warps take");
template <int EPW>
struct Smem {
    uint8_t a[Cfg<EPW>::STAGES][BM * BK];
    uint8_t b[Cfg<EPW>::STAGES][(BN / 2) * BK];
    uint64_t full[Cfg<EPW>::STAGES], empty[Cfg<EPW>::STAGES];
    uint64_t seg_full[2], seg_empty[2];
    uint32_t tmem_base;
    float qred[2][4];                          // OUTM 2: per (column half, row quarter) absmax
    alignas(1024) uint8_t stage_out[EPW][32 * 128];
    // EPW 8: second staging buffer per warp -- the TMA store of chunk c drains
    // while chunk c+1 is staged
    alignas(1024) uint8_t stage_out2[Cfg<EPW>::STG2 ? EPW : 1][32 * 128];
};
template <int EPW>
constexpr size_t smem_bytes() { return sizeof(Smem<EPW>) + 1024; }
static_assert(smem_bytes<8>() <= 232448 && smem_bytes<16>() <= 232448, "2-SM W8A8 shared memory over 227 KB");
}  // namespace gemm2

// Epilogue warps per mode: the exact promotion (three rounded ops per element,
// FMA-pipe heavy) gains 3-8% from 16 warps; the fast one (one FFMA2 per pair)
// loses 5-9% to the smaller ring and single-buffered staging 16 warps leave
// room for (same-box A/B, tools/ab_w8.sh)
#ifndef TB_W8_EPW_EXACT
#define TB_W8_EPW_EXACT 16
#endif
#ifndef TB_W8_EPW_FAST
#define TB_W8_EPW_FAST 8
#endif

// Tile raster of the 2-SM kernel: groups of W8_GROUP_M row-pair bands, row
// band fastest inside a group, so the ~74 co-running clusters share a few A
// bands and a few B column tiles (both L2-resident) instead of streaming every
// B tile once per A band.
#ifndef W8_GROUP_M
#define W8_GROUP_M 8
#endif
__device__ __forceinline__ void tile_coords(int tile, int nmp, int nnt, int &mp, int &nt) {
    const int per = W8_GROUP_M * nnt;
    const int g = tile / per, w = tile - g * per;
    const int m0 = g * W8_GROUP_M;
    const int gs = min(W8_GROUP_M, nmp - m0);
    mp = m0 + w % gs;
    nt = w / gs;
}

// Fused Ulysses forward exchange (planar bf16 output only): one tensor map per
// destination rank over that rank's head-shard buffer [3*hp, L, plane] (q, k, v
// planes of its hp heads, all L tokens).  Output plane c/plane = w*H + head
// (w = q/k/v) goes to rank head/hp, plane w*hp + head%hp, at global token row
// row0 + local row -- the GEMM's epilogue stores each tile straight into the
// head owner's buffer over peer memory, replacing the q/k/v all-to-all.
constexpr int MAX_PEERS = 8;
struct alignas(64) PeerMaps {
    CUtensorMap m[MAX_PEERS];
    int32_t n, hp, H, row0;
};

// OUTM: 0 f32, 1 bf16, 2 block-quantized INT8 (the next projection's A
// operand: the bf16-rounded result quantized per 128x128 block exactly like
// quantize_blockwise, codes TMA-stored, one f32 scale per block to qscales).
template <bool EXACT, int OUTM, int EPW>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(gemm2::Cfg<EPW>::THREADS, 1) w8a8_2sm_kernel(
    const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
    const __grid_constant__ CUtensorMap tma_out,
    const float *__restrict__ sa, const float *__restrict__ sb, const float *__restrict__ bias,
    int M, int N, int K, int plane, int act, float *__restrict__ qscales, const __grid_constant__ PeerMaps pm) {
    using namespace gemm2;
    using C = Cfg<EPW>;
    constexpr int STAGES = C::STAGES;
    constexpr bool OUT_BF16 = OUTM == 1;
    constexpr int CW = C::CW;
    static_assert(OUTM != 2 || EPW == 8, "the quantizing epilogue needs 8 epilogue warps (128-column halves)");
    constexpr uint32_t TMEM_COLS = 2 * BN;
    extern __shared__ uint8_t smem_raw[];
    Smem<EPW> &S = *reinterpret_cast<Smem<EPW> *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = ptx::cluster_ctarank();
    const int cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
    const int nmp = (M + 2 * BM - 1) / (2 * BM), nnt = N / BN, nkb = K / BK, nnb = N / 128;
    const int nmb = (M + 127) / 128;
    const int ntiles = nmp * nnt;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < STAGES; s++) { ptx::mbar_init(&S.full[s], 1); ptx::mbar_init(&S.empty[s], 1); }
        for (int b = 0; b < 2; b++) { ptx::mbar_init(&S.seg_full[b], 1); ptx::mbar_init(&S.seg_empty[b], 2 * EPW); }
        ptx::fence_barrier_init();
        ptx::prefetch_tmap(&tma_a);
        ptx::prefetch_tmap(&tma_b);
    }
    if (warp == 1) ptx::tmem_alloc_pair<TMEM_COLS>(&S.tmem_base);
    ptx::tc_fence_before();
    ptx::cluster_sync();                       // barriers of both CTAs initialised, TMEM allocated
    ptx::tc_fence_after();
    const uint32_t tmem = S.tmem_base;

    if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" :: "n"(C::CTRL_REGS));
    if (warp == 0) {
        if (ptx::elect_one()) {
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = cluster; tile < ntiles; tile += nclusters) {
                int mp, nt;
                tile_coords(tile, nmp, nnt, mp, nt);
                for (int kb = 0; kb < nkb; kb++) {
                    ptx::mbar_wait_sleep(&S.empty[stage], phase ^ 1);
                    const uint32_t fullc = ptx::mapa(ptx::smem_u32(&S.full[stage]), 0);
                    if (rank == 0) ptx::mbar_arrive_expect_tx(&S.full[stage], 2 * (BM + BN / 2) * BK);
                    ptx::tma_load_2d_pair(S.a[stage], &tma_a, kb * BK, mp * 2 * BM + (int)rank * BM, fullc);
                    ptx::tma_load_2d_pair(S.b[stage], &tma_b, kb * BK, nt * BN + (int)rank * (BN / 2), fullc);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (rank == 0) {
            int stage = 0, buf = 0;
            uint32_t phase = 0, bphase = 0;
            constexpr uint32_t idesc = ptx::idesc_i8(2 * BM, BN);
            for (int tile = cluster; tile < ntiles; tile += nclusters) {
                for (int kb = 0; kb < nkb; kb++) {
                    // segment buffer drained by both CTAs' epilogues; their initial
                    // arrive completes phase 0 before first use
                    ptx::mbar_wait_sleep(&S.seg_empty[buf], bphase);
                    ptx::mbar_wait_sleep(&S.full[stage], phase);
                    ptx::tc_fence_after();
                    const uint64_t ad = ptx::sdesc_sw128(ptx::smem_u32(S.a[stage]));
                    const uint64_t bd = ptx::sdesc_sw128(ptx::smem_u32(S.b[stage]));
                    if (ptx::elect_one()) {
#pragma unroll
                        for (int k = 0; k < BK / 32; k++)
                            ptx::mma_i8_pair(tmem + buf * BN, ad + 2 * k, bd + 2 * k, idesc, k > 0 ? 1u : 0u);
                        ptx::mma_commit_pair(&S.empty[stage], 0x3);
                        ptx::mma_commit_pair(&S.seg_full[buf], 0x3);
                    }
                    __syncwarp();
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                    buf ^= 1;
                    if (buf == 0) bphase ^= 1;
                }
            }
        }
    }
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" :: "n"(C::EPI_REGS));
        // warp index through a shuffle: provably warp-uniform, so the TMEM
        // addresses below live in uniform registers (no R2UR per tcgen05 op)
        const int wu = __shfl_sync(0xffffffffu, warp, 0);
        const int ew = wu - 4;
        const int quarter = wu & 3;                // TMEM lanes this warp may touch
        const int cg = ew >> 2;                    // column group of CW columns
        const uint32_t seg_empty0 = ptx::mapa(ptx::smem_u32(&S.seg_empty[0]), 0);
        const uint32_t seg_empty1 = ptx::mapa(ptx::smem_u32(&S.seg_empty[1]), 0);
        int buf = 0;
        uint32_t bphase = 0;
#pragma unroll
        for (int b = 0; b < 2; b++) {
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive_cluster(b ? seg_empty1 : seg_empty0);
        }
        for (int tile = cluster; tile < ntiles; tile += nclusters) {
            int mp, nt;
            tile_coords(tile, nmp, nnt, mp, nt);
            const int col0 = nt * BN + cg * CW;
            const int nb = col0 / 128;
            const int mb = 2 * mp + (int)rank;                    // this CTA's 128-row scale block
            const int mbs = mb < nmb ? mb : nmb - 1;              // (rows past M are clipped anyway)
            float2 acc2[CW / 2];
#pragma unroll
            for (int i = 0; i < CW / 2; i++) acc2[i] = make_float2(0.0f, 0.0f);
            // per-k-block scales by pointer walk (next k-block's pair prefetched)
            const float *pa = sa + (size_t)mbs * nkb, *pb = sb + nb;
            float s_a = __ldg(pa), s_b = __ldg(pb);
            for (int kb = 0; kb < nkb; kb++) {
                const float2 sa2 = make_float2(s_a, s_a), sb2 = make_float2(s_b, s_b);
                const float2 sab2 = make_float2(s_a * s_b, s_a * s_b);
                if (kb + 1 < nkb) {
                    pa += 1;
                    pb += nnb;
                    s_a = __ldg(pa);
                    s_b = __ldg(pb);
                }
                ptx::mbar_wait_sleep(&S.seg_full[buf], bphase);
                ptx::tc_fence_after();
                const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + buf * BN + cg * CW;
                auto promote = [&](const uint32_t *r, int c0, int n) {
#pragma unroll
                    for (int i = 0; i < n; i += 2) {
                        const float2 x = make_float2(__int2float_rn((int)r[i]), __int2float_rn((int)r[i + 1]));
                        float2 &o = acc2[(c0 + i) >> 1];
                        if constexpr (EXACT) {
                            // the reference sequence bit-for-bit: packed RN ops round each
                            // lane like the scalar op, but ptxas contracts a packed multiply
                            // feeding a packed add into FFMA2 (tools/ubench_f32x2.cu), so the
                            // product that feeds the add is formed with scalar RN multiplies
                            const float2 p = ptx::fmul2(x, sa2);
#if TB_W8_EXACT_FMA0
                            // p * sb as a packed FMA with a +0 addend: the RN product except
                            // that -0 becomes +0, which cannot change o (it starts at +0, and
                            // x + (+0) == x + (-0) for every x != -0); ptxas neither folds it
                            // into a multiply nor contracts it into the add
                            o = ptx::fadd2(o, ptx::ffma2(p, sb2, make_float2(0.0f, 0.0f)));
#else
                            o = ptx::fadd2(o, make_float2(__fmul_rn(p.x, sb2.x), __fmul_rn(p.y, sb2.y)));
#endif
                        } else {
                            o = ptx::ffma2(x, sab2, o);
                        }
                    }
                };
                if constexpr (EPW == 8) {
                    // 32-column groups, double-buffered: tcgen05.wait::ld covers every
                    // outstanding load, so group g+1's loads are issued before group g's math
                    constexpr int G = 32, NG = CW / G;
                    uint32_t rb[2][G];
                    ptx::tmem_ld16(taddr, *reinterpret_cast<uint32_t (*)[16]>(&rb[0][0]));
                    ptx::tmem_ld16(taddr + 16, *reinterpret_cast<uint32_t (*)[16]>(&rb[0][16]));
#pragma unroll
                    for (int g = 0; g < NG; g++) {
                        ptx::tmem_wait_ld();
                        if (g + 1 < NG) {
                            ptx::tmem_ld16(taddr + (g + 1) * G, *reinterpret_cast<uint32_t (*)[16]>(&rb[(g + 1) & 1][0]));
                            ptx::tmem_ld16(taddr + (g + 1) * G + 16,
                                           *reinterpret_cast<uint32_t (*)[16]>(&rb[(g + 1) & 1][16]));
                        }
                        promote(rb[g & 1], g * G, G);
                    }
                } else {
                    // 16-column groups, one in flight: the four warps of each SM
                    // sub-partition interleave their load / promote phases
                    constexpr int G = 16, NG = CW / G;
#pragma unroll
                    for (int g = 0; g < NG; g++) {
                        uint32_t r[G];
                        ptx::tmem_ld16(taddr + g * G, r);
                        ptx::tmem_wait_ld();
                        promote(r, g * G, G);
                    }
                }
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive_cluster(buf ? seg_empty1 : seg_empty0);   // the leader's barrier
                buf ^= 1;
                if (buf == 0) bphase ^= 1;
            }
            if (bias) {
#pragma unroll
                for (int i = 0; i < CW / 2; i++) {
                    acc2[i].x = __fadd_rn(acc2[i].x, __ldg(bias + col0 + 2 * i));
                    acc2[i].y = __fadd_rn(acc2[i].y, __ldg(bias + col0 + 2 * i + 1));
                }
            }
            if (act == 1) {
#pragma unroll
                for (int i = 0; i < CW / 2; i++) { acc2[i].x = gelu_tanh(acc2[i].x); acc2[i].y = gelu_tanh(acc2[i].y); }
            }
            const uint32_t stg_s = ptx::smem_u32(S.stage_out[ew]);
            const int row0 = mp * 2 * BM + (int)rank * BM + quarter * 32;
            if constexpr (OUTM == 2) {
                // block absmax of the bf16-rounded values (rows >= M excluded) over
                // the 4 row-quarter warps of this column half (named barrier per half)
                const int half = cg;
                const bool rok = row0 + lane < M;
                float am = 0.0f;
#pragma unroll
                for (int i = 0; i < CW / 2; i++) {
                    acc2[i].x = __bfloat162float(__float2bfloat16_rn(acc2[i].x));
                    acc2[i].y = __bfloat162float(__float2bfloat16_rn(acc2[i].y));
                    am = fmaxf(am, fmaxf(fabsf(acc2[i].x), fabsf(acc2[i].y)));
                }
                am = warp_max<32>(rok ? am : 0.0f);
                if (lane == 0) S.qred[half][quarter] = am;
                ptx::named_bar_sync(1 + half, 128);
                am = fmaxf(fmaxf(S.qred[half][0], S.qred[half][1]), fmaxf(S.qred[half][2], S.qred[half][3]));
                ptx::named_bar_sync(1 + half, 128);            // qred reusable
                const float sc = quant_scale(am);
                if (quarter == 0 && lane == 0 && mb < nmb) qscales[(int64_t)mb * nnb + nb] = sc;
                const float safe = (sc == 0.0f) ? 1.0f : sc;
                const float inv = __frcp_rn(safe);
                const bool exq = !(safe >= 1.17549435e-38f && inv <= 3.0e38f);   // subnormal scale: exact division
                if (lane == 0) ptx::bulk_wait_read0();
                __syncwarp();
#pragma unroll
                for (int u = 0; u < 8; u++) {                  // 16 codes (one 16-B unit) per step
                    float xv[16];
#pragma unroll
                    for (int j = 0; j < 8; j++) { xv[2 * j] = acc2[8 * u + j].x; xv[2 * j + 1] = acc2[8 * u + j].y; }
                    uint32_t w[4];
                    quant16_fast(xv, safe, inv, exq, w);
                    const uint32_t dst = stg_s + lane * 128 + ((u ^ (lane & 7)) * 16);
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" :: "r"(dst), "r"(w[0]), "r"(w[1]),
                                 "r"(w[2]), "r"(w[3]) : "memory");
                }
                ptx::fence_async_smem();
                __syncwarp();
                if (lane == 0) {
                    ptx::tma_store_2d(&tma_out, S.stage_out[ew], col0, row0);
                    ptx::bulk_commit();
                }
                continue;
            }
            constexpr int CPC = OUT_BF16 ? 64 : 32;             // columns per 128-B staged row
            static_assert(!C::STG2 || (CW / CPC) % 2 == 0, "chunk count per tile must be even");
#pragma unroll
            for (int ch = 0; ch < CW / CPC; ch++) {
                uint8_t *stg = (C::STG2 && (ch & 1)) ? S.stage_out2[C::STG2 ? ew : 0] : S.stage_out[ew];
                const uint32_t stg_c = ptx::smem_u32(stg);
                if (lane == 0) {
                    if (C::STG2) ptx::bulk_wait_read1();        // the store that last used this buffer has read it
                    else ptx::bulk_wait_read0();
                }
                __syncwarp();
#pragma unroll
                for (int u = 0; u < 8; u++) {
                    uint32_t w0, w1, w2, w3;
                    if constexpr (OUT_BF16) {
                        const int p = (ch * CPC + 8 * u) >> 1;
                        __nv_bfloat162 b0 = __floats2bfloat162_rn(acc2[p].x, acc2[p].y);
                        __nv_bfloat162 b1 = __floats2bfloat162_rn(acc2[p + 1].x, acc2[p + 1].y);
                        __nv_bfloat162 b2 = __floats2bfloat162_rn(acc2[p + 2].x, acc2[p + 2].y);
                        __nv_bfloat162 b3 = __floats2bfloat162_rn(acc2[p + 3].x, acc2[p + 3].y);
                        w0 = *reinterpret_cast<uint32_t *>(&b0); w1 = *reinterpret_cast<uint32_t *>(&b1);
                        w2 = *reinterpret_cast<uint32_t *>(&b2); w3 = *reinterpret_cast<uint32_t *>(&b3);
                    } else {
                        const int p = (ch * CPC + 4 * u) >> 1;
                        w0 = __float_as_uint(acc2[p].x); w1 = __float_as_uint(acc2[p].y);
                        w2 = __float_as_uint(acc2[p + 1].x); w3 = __float_as_uint(acc2[p + 1].y);
                    }
                    const uint32_t dst = stg_c + lane * 128 + ((u ^ (lane & 7)) * 16);
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" :: "r"(dst), "r"(w0), "r"(w1), "r"(w2),
                                 "r"(w3) : "memory");
                }
                ptx::fence_async_smem();
                __syncwarp();
                if (lane == 0) {
                    const int c = col0 + ch * CPC;
                    if (pm.n) {
                        // the head owner's buffer; boxes past this rank's rows are
                        // skipped (they would land in the next rank's token rows)
                        const int pl = c / plane, w = pl / pm.H, hd = pl - w * pm.H, owner = hd / pm.hp;
                        if (row0 < M)
                            ptx::tma_store_3d(&pm.m[owner], stg, c % plane, pm.row0 + row0,
                                              w * pm.hp + (hd - owner * pm.hp));
                    } else if (plane) {
                        ptx::tma_store_3d(&tma_out, stg, c % plane, row0, c / plane);
                    } else {
                        ptx::tma_store_2d(&tma_out, stg, c, row0);
                    }
                    ptx::bulk_commit();
                }
            }
            (void)stg_s;
        }
        if (lane == 0) ptx::bulk_wait_read0();
    }
    ptx::tc_fence_before();
    ptx::cluster_sync();                       // no CTA leaves while its peer may still signal it
    if (warp == 1) ptx::tmem_dealloc_pair<TMEM_COLS>(tmem);
}

// ------------------------------------------------------------ CUDA-core path
// Any block size / shape.  64x64 output tile per CTA, 256 threads x 4x4
// outputs, exact int32 segments via dp4a, identical promotion order.
__global__ void __launch_bounds__(256) w8a8_simt_kernel(const int8_t *__restrict__ a, const float *__restrict__ sa,
                                                        const int8_t *__restrict__ bt, const float *__restrict__ sb,
                                                        const float *__restrict__ bias, int64_t M, int64_t N,
                                                        int64_t K, int64_t block, int exact, void *out, int out_bf16) {
    __shared__ __align__(16) int8_t as_[64][68];
    __shared__ __align__(16) int8_t bs_[64][68];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int64_t m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
    const int64_t nkb = cdiv(K, block), nnb = cdiv(N, block);
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) acc[i][j] = 0.0f;
    for (int64_t kb = 0; kb < nkb; kb++) {
        const int64_t k0 = kb * block, k1 = min(k0 + block, K);
        int seg[4][4];
#pragma unroll
        for (int i = 0; i < 4; i++)
#pragma unroll
            for (int j = 0; j < 4; j++) seg[i][j] = 0;
        for (int64_t kc = k0; kc < k1; kc += 64) {
            __syncthreads();
            for (int i = threadIdx.x; i < 64 * 64; i += 256) {
                int r = i >> 6, c = i & 63;
                int64_t k = kc + c;
                as_[r][c] = (m0 + r < M && k < k1) ? a[(m0 + r) * K + k] : (int8_t)0;
                bs_[r][c] = (n0 + r < N && k < k1) ? bt[(n0 + r) * K + k] : (int8_t)0;
            }
            __syncthreads();
#pragma unroll 4
            for (int c = 0; c < 64; c += 4) {
                int av[4], bv[4];
#pragma unroll
                for (int i = 0; i < 4; i++) av[i] = *reinterpret_cast<const int *>(&as_[ty * 4 + i][c]);
#pragma unroll
                for (int j = 0; j < 4; j++) bv[j] = *reinterpret_cast<const int *>(&bs_[tx * 4 + j][c]);
#pragma unroll
                for (int i = 0; i < 4; i++)
#pragma unroll
                    for (int j = 0; j < 4; j++) seg[i][j] = __dp4a(av[i], bv[j], seg[i][j]);
            }
        }
#pragma unroll
        for (int i = 0; i < 4; i++) {
            const int64_t m = m0 + ty * 4 + i;
            const float ra = (m < M) ? sa[(m / block) * nkb + kb] : 0.0f;
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const int64_t n = n0 + tx * 4 + j;
                const float cb = (n < N) ? sb[kb * nnb + n / block] : 0.0f;
                const float v = (float)seg[i][j];
                acc[i][j] = exact ? __fadd_rn(acc[i][j], __fmul_rn(__fmul_rn(v, ra), cb)) : fmaf(v, ra * cb, acc[i][j]);
            }
        }
    }
#pragma unroll
    for (int i = 0; i < 4; i++) {
        const int64_t m = m0 + ty * 4 + i;
        if (m >= M) continue;
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const int64_t n = n0 + tx * 4 + j;
            if (n >= N) continue;
            float v = bias ? __fadd_rn(acc[i][j], bias[n]) : acc[i][j];
            if (out_bf16) reinterpret_cast<__nv_bfloat16 *>(out)[m * N + n] = __float2bfloat16_rn(v);
            else reinterpret_cast<float *>(out)[m * N + n] = v;
        }
    }
}

static int g_num_sms = 0;
int num_sms() {
    if (!g_num_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms <= 0) g_num_sms = 148;
    }
    return g_num_sms;
}

int w8a8_dispatch(const int8_t *a, const float *sa, const int8_t *bt, const float *sb, const float *bias,
                  int64_t M, int64_t N, int64_t K, int64_t block, void *out, int out_dtype, int exact,
                  cudaStream_t st, int64_t plane = 0, int act = 0) {
    TB_REQUIRE(plane == 0 || (plane > 0 && 128 % plane == 0 && N % plane == 0 && out_dtype == TB_BF16 && plane >= 64),
               "plane must divide 128 and N, be >= 64, with bf16 output");
    TB_REQUIRE(act == 0 || act == 1, "act must be 0 (none) or 1 (gelu-tanh)");
    TB_REQUIRE(block >= 1, "block must be >= 1");
    // segments accumulate exactly in int32 (tensor cores: s32 TMEM; SIMT: dp4a)
    // and are rounded to f32 once, like the reference's int64 path above its
    // f32-exact bound of 1040 (blockquant.py:26,119-129): exact while
    // block * 127^2 < 2^31
    TB_REQUIRE(block * 16129 < (1ll << 31), "block edge too large for an exact int32 segment (block * 127^2 >= 2^31)");
    TB_REQUIRE(out_dtype == TB_F32 || out_dtype == TB_BF16, "out dtype must be f32 or bf16");
    if (M == 0 || N == 0) return TB_OK;
    const bool tc = block == 128 && K % 128 == 0 && N % 128 == 0 && K > 0 && M < (1ll << 31) &&
                    ((uintptr_t)a % 16) == 0 && ((uintptr_t)bt % 16) == 0 && ((uintptr_t)out % 16) == 0;
    // 2-SM kernel (CTA pairs, 256x256 tiles, register-rebalanced epilogue) by
    // default where the shape allows; TB_W8A8_2SM=0 forces the 1-SM kernel
    static const bool use2sm = [] { const char *e = getenv("TB_W8A8_2SM"); return !e || atoi(e) != 0; }();
    if (tc && use2sm && N % 256 == 0 && M >= 256) {
        CUtensorMap ta, tbm, tout;
        const bool obf = out_dtype == TB_BF16;
        bool okm = make_tmap_2d(&ta, a, CU_TENSOR_MAP_DATA_TYPE_UINT8, K, M, K, 128, 128) &&
                   make_tmap_2d(&tbm, bt, CU_TENSOR_MAP_DATA_TYPE_UINT8, K, N, K, 128, 128);
        if (plane)       // planes [N/plane][M][plane] (bf16), box 64 columns x 32 rows
            okm = okm && make_tmap_3d(&tout, out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, plane, M, N / plane, plane * 2,
                                      M * plane * 2, 64, 32, 1);
        else
            okm = okm && make_tmap_2d(&tout, out, obf ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                                      N, M, N * (obf ? 2 : 4), obf ? 64 : 32, 32);
        if (!okm) return fail(TB_ECUDA, "cuTensorMapEncodeTiled failed");
        const int ntiles = (int)(cdiv(M, 256) * (N / 256));
        int clusters = num_sms() / 2;
        if (ntiles < clusters) clusters = ntiles;
        const int grid = 2 * clusters;
        PeerMaps no_peers;
        memset(&no_peers, 0, sizeof(no_peers));
#define TB_GEMM2(E, B)                                                                                     \
    {                                                                                                      \
        constexpr int EPW = (E) ? TB_W8_EPW_EXACT : TB_W8_EPW_FAST;                                       \
        auto kern = w8a8_2sm_kernel<E, (B) ? 1 : 0, EPW>;                                                  \
        smem_attr(kern, (int)gemm2::smem_bytes<EPW>());                                                    \
        kern<<<grid, gemm2::Cfg<EPW>::THREADS, gemm2::smem_bytes<EPW>(), st>>>(                            \
            ta, tbm, tout, sa, sb, bias, (int)M, (int)N, (int)K,                                           \
                                                              (int)plane, act, nullptr, no_peers);               \
    }
        if (exact && !obf) TB_GEMM2(true, false)
        else if (exact) TB_GEMM2(true, true)
        else if (!obf) TB_GEMM2(false, false)
        else TB_GEMM2(false, true)
#undef TB_GEMM2
        return check_launch("w8a8_2sm");
    }
    if (tc) {
        const int BN = (N % 256 == 0) ? 256 : 128;
        CUtensorMap ta, tbm;
        CUtensorMap tout;
        const bool obf = out_dtype == TB_BF16;
        bool okm = make_tmap_2d(&ta, a, CU_TENSOR_MAP_DATA_TYPE_UINT8, K, M, K, 128, 128) &&
                   make_tmap_2d(&tbm, bt, CU_TENSOR_MAP_DATA_TYPE_UINT8, K, N, K, 128, BN);
        if (plane)       // planes [N/plane][M][plane] (bf16), box 64 columns x 32 rows
            okm = okm && make_tmap_3d(&tout, out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, plane, M, N / plane, plane * 2,
                                      M * plane * 2, 64, 32, 1);
        else
            okm = okm && make_tmap_2d(&tout, out, obf ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                                      N, M, N * (obf ? 2 : 4), obf ? 64 : 32, 32);
        if (!okm) return fail(TB_ECUDA, "cuTensorMapEncodeTiled failed");
        const int ntiles = (int)(cdiv(M, 128) * (N / BN));
        const int grid = ntiles < num_sms() ? ntiles : num_sms();
#define TB_GEMM_LAUNCH(BNV, E, B)                                                                          \
    {                                                                                                      \
        auto kern = w8a8_tc_kernel<BNV, E, B>;                                                             \
        smem_attr(kern, (int)gemm::smem_bytes<BNV>()); \
        kern<<<grid, gemm::THREADS, gemm::smem_bytes<BNV>(), st>>>(ta, tbm, tout, sa, sb, bias, out, (int)M, (int)N, (int)K, \
                                                                  (int)plane, act);                                        \
    }
#define TB_GEMM_BN(BNV)                                                                                    \
        if (exact && out_dtype == TB_F32) TB_GEMM_LAUNCH(BNV, true, false)                                 \
        else if (exact) TB_GEMM_LAUNCH(BNV, true, true)                                                    \
        else if (out_dtype == TB_F32) TB_GEMM_LAUNCH(BNV, false, false)                                    \
        else TB_GEMM_LAUNCH(BNV, false, true)
        if (BN == 256) { TB_GEMM_BN(256) } else { TB_GEMM_BN(128) }
#undef TB_GEMM_BN
#undef TB_GEMM_LAUNCH
        return check_launch("w8a8_tc");
    }
    TB_REQUIRE(plane == 0 && act == 0, "planar output / fused activation need the tensor-core path");
    dim3 grid((unsigned)cdiv(N, 64), (unsigned)cdiv(M, 64));
    w8a8_simt_kernel<<<grid, 256, 0, st>>>(a, sa, bt, sb, bias, M, N, K, block, exact, out, out_dtype == TB_BF16);
    return check_launch("w8a8_simt");
}

}  // namespace tb

using namespace tb;

extern "C" int tb_w8a8_gemm(const int8_t *a, const float *sa, const int8_t *bt, const float *sb, const float *bias,
                            int64_t M, int64_t N, int64_t K, int64_t block, void *out, int out_dtype, void *stream) {
    return w8a8_dispatch(a, sa, bt, sb, bias, M, N, K, block, out, out_dtype, 1, as_stream(stream));
}

extern "C" int tb_w8a8_gemm_fast(const int8_t *a, const float *sa, const int8_t *bt, const float *sb,
                                 const float *bias, int64_t M, int64_t N, int64_t K, int64_t block, void *out,
                                 int out_dtype, void *stream) {
    return w8a8_dispatch(a, sa, bt, sb, bias, M, N, K, block, out, out_dtype, 0, as_stream(stream));
}

extern "C" int tb_quantized_linear(const void *x, int x_dtype, const int8_t *bt, const float *sb, const float *bias,
                                   int64_t M, int64_t N, int64_t K, int64_t block, int8_t *xq_ws, float *xs_ws,
                                   void *out, int out_dtype, void *stream) {
    int rc = tb_quantize_blockwise(x, x_dtype, M, K, block, xq_ws, xs_ws, nullptr, stream);
    if (rc) return rc;
    return tb_w8a8_gemm(xq_ws, xs_ws, bt, sb, bias, M, N, K, block, out, out_dtype, stream);
}

extern "C" int tb_w8a8_gemm_fast_ex(const int8_t *a, const float *sa, const int8_t *bt, const float *sb,
                                    const float *bias, int64_t M, int64_t N, int64_t K, int64_t block, void *out,
                                    int out_dtype, int64_t plane, int act, void *stream) {
    return w8a8_dispatch(a, sa, bt, sb, bias, M, N, K, block, out, out_dtype, 0, as_stream(stream), plane, act);
}

// Fast-mode GEMM whose epilogue block-quantizes its (bf16-rounded, optionally
// GELU'd) result for the next projection: codes [M, N] int8 row-major and
// scales [ceil(M/128), N/128] f32, bit-identical to tb_quantize_blockwise of
// the bf16 output of tb_w8a8_gemm_fast_ex.  2-SM kernel shapes only
// (N % 256 == 0, M >= 256, K % 128 == 0); TB_EUNSUPPORTED otherwise.
extern "C" int tb_w8a8_gemm_quant(const int8_t *a, const float *sa, const int8_t *bt, const float *sb,
                                  const float *bias, int64_t M, int64_t N, int64_t K, int64_t block, int act,
                                  int8_t *q_out, float *scales_out, void *stream) {
    TB_REQUIRE(act == 0 || act == 1, "act must be 0 (none) or 1 (gelu-tanh)");
    if (M == 0 || N == 0) return TB_OK;
    const bool ok = block == 128 && K % 128 == 0 && K > 0 && N % 256 == 0 && M >= 256 && M < (1ll << 31) &&
                    ((uintptr_t)a % 16) == 0 && ((uintptr_t)bt % 16) == 0 && ((uintptr_t)q_out % 16) == 0;
    if (!ok) return fail(TB_EUNSUPPORTED, "quantizing epilogue needs block 128, N % 256 == 0, M >= 256");
    CUtensorMap ta, tbm, tout;
    if (!make_tmap_2d(&ta, a, CU_TENSOR_MAP_DATA_TYPE_UINT8, K, M, K, 128, 128) ||
        !make_tmap_2d(&tbm, bt, CU_TENSOR_MAP_DATA_TYPE_UINT8, K, N, K, 128, 128) ||
        !make_tmap_2d(&tout, q_out, CU_TENSOR_MAP_DATA_TYPE_UINT8, N, M, N, 128, 32))
        return fail(TB_ECUDA, "cuTensorMapEncodeTiled failed");
    const int ntiles = (int)(cdiv(M, 256) * (N / 256));
    int clusters = num_sms() / 2;
    if (ntiles < clusters) clusters = ntiles;
    auto kern = w8a8_2sm_kernel<false, 2, 8>;
    smem_attr(kern, (int)gemm2::smem_bytes<8>());
    PeerMaps no_peers;
    memset(&no_peers, 0, sizeof(no_peers));
    kern<<<2 * clusters, gemm2::Cfg<8>::THREADS, gemm2::smem_bytes<8>(), as_stream(stream)>>>(
        ta, tbm, tout, sa, sb, bias, (int)M, (int)N, (int)K, 0, act, scales_out, no_peers);
    return check_launch("w8a8_gemm_quant");
}

// Fused Ulysses forward exchange: the qkv projection of this rank's token shard
// (rows [row0, row0 + M) of the sequence) with every 64-column x 32-row output
// box TMA-stored into the head owner's buffer.  peers: HOST array of P device
// pointers (peer memory), each bf16 [3*hp, L, 128] (q, k, v planes of that
// rank's hp = H/P heads); N = 3*H*128; 2-SM kernel shapes (M >= 256).
extern "C" int tb_w8a8_gemm_qkv_peers(const int8_t *a, const float *sa, const int8_t *bt, const float *sb,
                                      const float *bias, int64_t M, int64_t N, int64_t K, int64_t block,
                                      void *const *peers, int64_t P, int64_t H, int64_t row0, int64_t L,
                                      void *stream) {
    TB_REQUIRE(peers != nullptr && P >= 1 && P <= MAX_PEERS && H % P == 0, "1 <= P <= 8 peers, H % P == 0");
    TB_REQUIRE(N == 3 * H * 128, "N must be 3 * H * 128 (q, k, v planes of 128)");
    TB_REQUIRE(row0 >= 0 && row0 + M <= L, "token rows out of range");
    if (M == 0) return TB_OK;
    const bool ok = block == 128 && K % 128 == 0 && K > 0 && N % 256 == 0 && M >= 256 && M < (1ll << 31) &&
                    ((uintptr_t)a % 16) == 0 && ((uintptr_t)bt % 16) == 0;
    if (!ok) return fail(TB_EUNSUPPORTED, "peer qkv epilogue needs the 2-SM kernel shape (block 128, M >= 256)");
    const int64_t hp = H / P;
    CUtensorMap ta, tbm;
    PeerMaps pm;
    memset(&pm, 0, sizeof(pm));
    bool okm = make_tmap_2d(&ta, a, CU_TENSOR_MAP_DATA_TYPE_UINT8, K, M, K, 128, 128) &&
               make_tmap_2d(&tbm, bt, CU_TENSOR_MAP_DATA_TYPE_UINT8, K, N, K, 128, 128);
    for (int64_t r = 0; r < P; r++) {
        TB_REQUIRE(peers[r] != nullptr && (uintptr_t)peers[r] % 16 == 0, "peer buffers must be 16-B aligned");
        okm = okm && make_tmap_3d(&pm.m[r], peers[r], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 128, L, 3 * hp, 256,
                                  L * 256, 64, 32, 1);
    }
    if (!okm) return fail(TB_ECUDA, "cuTensorMapEncodeTiled failed (peers)");
    pm.n = (int)P; pm.hp = (int)hp; pm.H = (int)H; pm.row0 = (int)row0;
    const int ntiles = (int)(cdiv(M, 256) * (N / 256));
    int clusters = num_sms() / 2;
    if (ntiles < clusters) clusters = ntiles;
    auto kern = w8a8_2sm_kernel<false, 1, TB_W8_EPW_FAST>;
    smem_attr(kern, (int)gemm2::smem_bytes<TB_W8_EPW_FAST>());
    kern<<<2 * clusters, gemm2::Cfg<TB_W8_EPW_FAST>::THREADS, gemm2::smem_bytes<TB_W8_EPW_FAST>(),
           as_stream(stream)>>>(
        ta, tbm, ta, sa, sb, bias, (int)M, (int)N, (int)K, 128, 0, nullptr, pm);
    return check_launch("w8a8_gemm_qkv_peers");
}

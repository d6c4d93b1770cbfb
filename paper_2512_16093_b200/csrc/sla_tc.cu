// sla_tc.cu -- fused SLA + Sage block-sparse attention on tcgen05 (sm_100a).
//
// Replaces _sparse_branch (attention.py:347-389) and the combine of
// sla_attention (attention.py:410-421) for the throughput envelope
// (head_dim 128, q_block 128, kv_block 64, quantized INT8 branch).
//
// One CTA per (head, 128-row q-block); two CTAs per SM so one CTA's softmax
// overlaps the other's tensor-core work.  Warp roles (192 threads):
//   warps 0-3  softmax/epilogue, thread = query row = TMEM lane
//   warp 4     TMA producer: Q codes once; per selected kv block the K code
//              tile (64x128 int8) into a 3-stage ring (128B swizzle,
//              mbarrier complete_tx)
//   warp 6     TMA producer: per selected kv block the V tile (64 tokens x
//              128 channels bf16, two SW128 boxes) into its own 3-stage ring,
//              so K runs ahead of V
//   warp 5     MMA issuer (one elected thread):
//                S_j  = Qc . Kc_j^T   4 x tcgen05.mma kind::i8  (M128 N64 K32) -> s32 TMEM
//                O   += P_j . V_j     4 x tcgen05.mma kind::f16 (M128 N128 K16), A = P_j in TMEM
//              issued as QK(j+1) before PV(j) so QK overlaps softmax(j).
// TMEM (256 cols): two 64-col S buffers; P_j (bf16, 2 per column, 32 cols)
// overwrites S_j in place (FA4-style), so PV reads A straight from TMEM and
// the tensor pipe's in-order execution protects the S/P buffer reuse; O is
// the f32 accumulator in cols 128-255.
// Softmax per block (log2 domain): logit2 = s32 * (sq*sk*scale*log2e) +
// corr*scale*log2e with corr = q_row . k_mean; running reference max with
// lazy O rescaling (only when the block max exceeds it by > 8, i.e. p <=
// 256).  Epilogue: O and l rebased to the true row max, combined with the
// linear branch exactly as attention.py:416-421.
#include <cstdlib>
#include <type_traits>

#include <cuda_fp8.h>

#include "common.cuh"
#include "ptx.cuh"
#include "tmap.cuh"

namespace tb {

#ifndef TB_SLA_PP
#define TB_SLA_PP 0x52
#endif
// TB_SLA_BIAS: seed each S tile with the float bits of 1.5*2^23 through one
// kind::f16 MMA, so the s32 scores come out of TMEM already as the floats
// M + s (no per-element integer add in the softmax)
#ifndef TB_SLA_UNI
#define TB_SLA_UNI 1
#endif
// TB_SLA_EARLY: linear-first (non-Q2) tiles keep phi(Q) in TMEM (the second S
// buffer's columns) and KV_sel^T in v[0] + k[0..1] only, so the K / V
// producers start at once (rings offset past the staging slots) and QK(0)
// runs under the softmax warps' prologue
#ifndef TB_SLA_EARLY
#define TB_SLA_EARLY 1
#endif
#ifndef TB_SLA_BIAS
#define TB_SLA_BIAS 1
#endif

namespace sla {
// MMA-warp barrier waits: 0 = try_wait with suspend hint, 1 = try_wait, 2 = test_wait poll
#ifndef TB_SLA_MMA_WAIT
#define TB_SLA_MMA_WAIT 0
#endif
#if TB_SLA_MMA_WAIT == 0
#define MMA_WAIT ptx::mbar_wait_sleep
#elif TB_SLA_MMA_WAIT == 1
#define MMA_WAIT ptx::mbar_wait
#else
#define MMA_WAIT ptx::mbar_wait_spin
#endif
#ifndef TB_SLA_SM_SPIN
#define TB_SLA_SM_SPIN 0
#endif
#if TB_SLA_SM_SPIN
#define SM_WAIT ptx::mbar_wait_spin
#else
#define SM_WAIT ptx::mbar_wait_sleep
#endif
#ifndef TB_SLA_KST
#define TB_SLA_KST 3
#endif
constexpr int BM = 128, BN = 64, D = 128, KSTAGES = TB_SLA_KST, VSTAGES = 3;
// TB_SLA_REGS: a fourth (idle) control warp completes warpgroup 1, so
// setmaxnreg can move its registers to the softmax warpgroup: 64 per control
// thread, 192 per softmax thread (2 CTAs x 256 threads x 128 at launch).
// Measured 8.5 vs 8.95 ms at cfg4 (interleaved A/B, tools/ab_sla.sh)
#ifndef TB_SLA_REGS
#define TB_SLA_REGS 1
#endif
constexpr int THREADS = TB_SLA_REGS ? 256 : 224;   // 4 softmax + K producer + MMA + V producer (+ idle) warps
#ifndef TB_SLA_CTRL_REGS
#define TB_SLA_CTRL_REGS 64
#endif
#ifndef TB_SLA_SETMAXNREG
#define TB_SLA_SETMAXNREG 1
#endif
constexpr int CTRL_REGS = TB_SLA_CTRL_REGS, SOFTMAX_REGS = 128 + (128 - TB_SLA_CTRL_REGS);
static_assert(!TB_SLA_REGS || 128 * (128 - CTRL_REGS) >= 128 * (SOFTMAX_REGS - 128), "setmaxnreg budget");
constexpr uint32_t Q_BYTES = BM * D;          // int8
constexpr uint32_t K_BYTES = BN * D;          // int8
constexpr uint32_t V_BYTES = D * BN * 2;      // bf16 V tile: two 64-channel x 64-token SW128 boxes
// Q2 (q_block 64): the 128-row tile holds two 64-row q-blocks.  Its linear
// branch stages phi(Q) (32 KB) and both q-blocks' KV_sel^T (2 x 32 KB) in q..x
// (96 KB contiguous), so the tail x extends the rings by 8 KB.
constexpr uint32_t X_BYTES = 96 * 1024 - (Q_BYTES + 3 * V_BYTES + KSTAGES * K_BYTES);
static_assert(KSTAGES != 3 || X_BYTES == 8192, "Q2 staging layout assumes 3 K stages");
template <bool Q2>
struct SmemT {
    uint8_t q[Q_BYTES];
    uint8_t v[VSTAGES][V_BYTES];
    uint8_t k[KSTAGES][K_BYTES];
    uint8_t x[Q2 ? X_BYTES : 16];
    uint64_t q_full, o_final;
    uint64_t k_full[KSTAGES], k_empty[KSTAGES];
    uint64_t v_full[VSTAGES], v_empty[VSTAGES];
    uint64_t s_full[2], p_full[2], pv_done[2];
    uint64_t phiq_full, lin_full, lin_done;     // fused linear-branch epilogue
    uint64_t k1_full;                           // den row of KV_sel (sum phi(K_b) over the complement)
    uint64_t lin_fix, lin_done2;                // Q2: per-half hand-off of the linear numerator
    alignas(128) uint16_t bias_a[128], bias_b[128];  // bias-MMA operands (2 core matrices each)
    alignas(16) __nv_bfloat16 k1[Q2 ? 2 : 1][128];
    float corr_s[128], den_s[128];              // prologue: per-row q . k_mean and den_L
    float c1[2048];                             // per selected block: sq * sk * scale * log2e (Q2: sk * scale * log2e)
    uint8_t rag[2048];                          // per selected block: bit 2 ragged last kv block; Q2: bits 0/1 = q-halves
    uint32_t tmem_base;
};
template <bool Q2>
constexpr int max_sel() { return 2048; }
constexpr int MAX_SEL = 2048;                  // selected kv blocks per q-block (c1 / ragged tables)
constexpr float LOG2E = 1.4426950408889634f;
constexpr float LN2 = 0.6931471805599453f;
}  // namespace sla

#ifdef TB_SLA_TRACE
// diagnostic timestamps (clock64) of one CTA: [block][event]
__device__ unsigned long long tb_sla_trace[80][16];
// whole-launch phase accounting: [0..2] summed prologue / main loop / epilogue
// cycles of thread 0 over all CTAs, [3] CTA count; per SM: min entry / max exit
// clock64 and %globaltimer (ns)
__device__ unsigned long long tb_sla_phase[4];
__device__ unsigned long long tb_sla_sm[160][4];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void tb_phase_done(unsigned long long t0, unsigned long long g0, unsigned long long t1,
                                              unsigned long long t2) {
    const unsigned long long t3 = clock64(), g3 = gtimer();
    atomicAdd(&tb_sla_phase[0], t1 - t0);
    atomicAdd(&tb_sla_phase[1], t2 - t1);
    atomicAdd(&tb_sla_phase[2], t3 - t2);
    atomicAdd(&tb_sla_phase[3], 1ull);
    uint32_t sm;
    asm volatile("mov.u32 %0, %smid;" : "=r"(sm));
    atomicMin(&tb_sla_sm[sm][0], t0);
    atomicMax(&tb_sla_sm[sm][1], t3);
    atomicMin(&tb_sla_sm[sm][2], g0);
    atomicMax(&tb_sla_sm[sm][3], g3);
}
#define TB_PH(x) x
#define TB_TRACE(j, e)                                                                                   \
    do {                                                                                                 \
        if (blockIdx.x == 100 && blockIdx.y == 5 && (j) < 64) tb_sla_trace[(j)][(e)] = clock64();        \
    } while (0)
// rows 64.. : one-off events (prologue 70, epilogue 71)
#define TB_TRACE_X(row, e)                                                                               \
    do {                                                                                                 \
        if (blockIdx.x == 100 && blockIdx.y == 5) tb_sla_trace[(row)][(e)] = clock64();                  \
    } while (0)
#else
#define TB_TRACE(j, e) do {} while (0)
#define TB_TRACE_X(row, e) do {} while (0)
#define TB_PH(x) do {} while (0)
#endif

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// 2^x on the FMA/ALU pipes (FA4-style MUFU offload): round-to-nearest split
// x = j + f, f in [-0.5, 0.5], degree-3 minimax for 2^f (rel err 7.7e-5, well
// under the bf16 rounding of P), exponent added with one LEA.
__device__ __forceinline__ float ex2_poly(float x) {
    x = fmaxf(x, -126.0f);
    const float t = __fadd_rn(x, 12582912.0f);           // low bits = round(x)
    const float f = __fsub_rn(x, __fsub_rn(t, 12582912.0f));
    const float p = fmaf(fmaf(fmaf(0.055088773f, f, 0.24260406f), f, 0.69327623f), f, 0.99992895f);
    return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

// Packed form for two exponents: FFMA2/FADD2 carry the split and the Horner
// chain, so one pair costs ~10 issue slots and no MUFU/XU cycles.
__device__ __forceinline__ float2 ex2_poly2(float2 x) {
    x.x = fmaxf(x.x, -126.0f);
    x.y = fmaxf(x.y, -126.0f);
    const float2 M = make_float2(12582912.0f, 12582912.0f), NM = make_float2(-12582912.0f, -12582912.0f);
    const float2 t = ptx::fadd2(x, M);                                    // low mantissa bits = round(x)
    const float2 f = ptx::ffma2(ptx::fadd2(t, NM), make_float2(-1.0f, -1.0f), x);   // x - round(x)
    float2 p = ptx::ffma2(make_float2(0.055088773f, 0.055088773f), f, make_float2(0.24260406f, 0.24260406f));
    p = ptx::ffma2(p, f, make_float2(0.69327623f, 0.69327623f));
    p = ptx::ffma2(p, f, make_float2(0.99992895f, 0.99992895f));
    return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                       __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

// 2^y for two exponents entirely on the FMA pipe, from u = sat(y/256 + 125/256)
// (one saturating FFMA2 computes u from the score, so the clamp of y to
// [-125, 131] is free): t = M + round(y_c) with y_c = 256u - 125, f = y_c -
// round(y_c) in [-0.5, 0.5], degree-3 minimax for 2^f (rel err 7.7e-5, far
// under the bf16 rounding of P), exponent added with one integer op.  y_c >
// 127 gives inf/NaN, which the caller's row-sum check rejects.
__device__ __forceinline__ float2 ex2_poly2_sat(float2 u) {
    const float2 C = make_float2(12582912.0f - 125.0f, 12582912.0f - 125.0f);
    const float2 S256 = make_float2(256.0f, 256.0f);
    const float2 t = ptx::ffma2(u, S256, C);                                  // M + round(y_c)
    const float2 w = ptx::ffma2(t, make_float2(-1.0f, -1.0f), C);            // -round(y_c) - 125 (exact)
    const float2 f = ptx::ffma2(u, S256, w);                                  // y_c - round(y_c)
    float2 p = ptx::ffma2(make_float2(0.055088773f, 0.055088773f), f, make_float2(0.24260406f, 0.24260406f));
    p = ptx::ffma2(p, f, make_float2(0.69327623f, 0.69327623f));
    p = ptx::ffma2(p, f, make_float2(0.99992895f, 0.99992895f));
    return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                       __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

template <typename T>
__device__ __forceinline__ void load8(const T *p, float *x) {
    if constexpr (sizeof(T) == 2) {
        const uint4 w = *reinterpret_cast<const uint4 *>(p);
        const __nv_bfloat162 *b = reinterpret_cast<const __nv_bfloat162 *>(&w);
#pragma unroll
        for (int i = 0; i < 4; i++) { const float2 f = __bfloat1622float2(b[i]); x[2 * i] = f.x; x[2 * i + 1] = f.y; }
    } else {
        const float4 a = *reinterpret_cast<const float4 *>(p), b = *reinterpret_cast<const float4 *>(p + 4);
        x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w; x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
    }
}

// F8 (opt-in): P and V as e4m3 and PV as kind::f8f6f4
// (M128 N128 K32, A = P in TMEM, four per column; B = the V code tile, one
// 128-channel SW128 box, MN-major).  V carries one scale per head (oracle/
// oracle.py quantize_v_fp8); P is stored unscaled (p <= 448 is guaranteed: the
// fast path accepts a block only when its row sum is <= 448, the exact path
// rebases when the max outgrows the reference by > 8, i.e. p <= 256).  O
// accumulates sum p * v / sv; the fused linear numerator is brought to the
// same scale by staging phi(Q) / sv, and the epilogue multiplies by sv.
//
// Q2 (q_block 64, the reference default): the 128-row tile n holds q-blocks
// 2n (rows 0-63, warps 0-1) and 2n+1 (rows 64-127, warps 2-3).  The kernel
// walks the UNION of their top-k lists (tb_pair_union: ascending, entry =
// block | mask << 28) and a warp whose q-block did not select a block stores
// P = 0 for it, so each row attends exactly its own selection; Q scales, logit
// slopes and the linear branch's KV_sel / den row are per q-block.
template <typename T, bool EXACT, bool F8 = false, bool Q2 = false>
__global__ void __launch_bounds__(sla::THREADS, 2) sla_tc_kernel(
    const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
    const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_kv, tb_sla_args a, int nq,
    int nkv) {
    using namespace sla;
    using Smem = SmemT<Q2>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    Smem &S = *reinterpret_cast<Smem *>(smem_raw);    // dynamic smem starts 1024-aligned (no static smem)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n = blockIdx.x, h = blockIdx.y;
    const int count = (int)a.count;                 // per q-block (attention.py:279)
    const int L = (int)a.L;
    const int ntile = gridDim.x;
    // selected kv blocks this tile visits: the q-block's own list, or (Q2) the pair union
    const int nsel = Q2 ? __ldg(a.pair_cnt + (int64_t)h * ntile + n) : count;
    const int32_t *sel = Q2 ? a.pair_idx + ((int64_t)h * ntile + n) * a.pair_ld
                            : a.idx + ((int64_t)h * nq + n) * count;
    // q-block of each half of the tile (Q2: the second one may be past the sequence)
    const int qb0 = Q2 ? 2 * n : n;
    const int qb1 = Q2 ? (2 * n + 1 < nq ? 2 * n + 1 : 2 * n) : n;

#ifdef TB_SLA_TRACE
    unsigned long long ph_t0 = clock64(), ph_g0 = gtimer(), ph_t1 = 0, ph_t2 = 0;
#endif
    if (threadIdx.x == 0) TB_TRACE_X(70, 0);
    // softmax threads: their q row is pulled into L2 before the setup barrier,
    // so the DRAM latency overlaps barrier init / TMEM alloc
    if (warp < 4 && n * BM + (int)threadIdx.x < L) {
        const char *src = reinterpret_cast<const char *>(reinterpret_cast<const T *>(a.q) +
                                                         ((int64_t)h * L + n * BM + threadIdx.x) * D);
#pragma unroll
        for (int c = 0; c < (int)(D * sizeof(T)); c += 128) asm volatile("prefetch.global.L2 [%0];" :: "l"(src + c));
    }
    if (warp == 6) {
        // bias-MMA operands: A rows [1, 0 x7 | 1, 0 x7], B rows [M/2, 0 x7 | M/2, 0 x7]
#pragma unroll
        for (int i = lane; i < 128; i += 32) {
            S.bias_a[i] = (i % 8 == 0) ? 0x3F80 : 0;    // bf16 1.0
            S.bias_b[i] = (i % 8 == 0) ? 0x4AC0 : 0;    // bf16 6291456 = 1.5 * 2^22
        }
        ptx::fence_async_smem();
    }
    if (warp == 4 && lane == 0) {
        if (ptx::smem_u32(smem_raw) & 1023) __trap();     // SW128 tiles need 1024-B alignment
        ptx::mbar_init(&S.q_full, 1);
        ptx::mbar_init(&S.o_final, 1);
        for (int s = 0; s < KSTAGES; s++) { ptx::mbar_init(&S.k_full[s], 1); ptx::mbar_init(&S.k_empty[s], 1); }
        for (int s = 0; s < VSTAGES; s++) { ptx::mbar_init(&S.v_full[s], 1); ptx::mbar_init(&S.v_empty[s], 1); }
        for (int b = 0; b < 2; b++) {
            ptx::mbar_init(&S.s_full[b], 1);
            ptx::mbar_init(&S.p_full[b], 128);
            ptx::mbar_init(&S.pv_done[b], 1);
        }
        ptx::mbar_init(&S.lin_fix, 64);
        ptx::mbar_init(&S.lin_done2, 1);
        ptx::mbar_init(&S.phiq_full, 128);
        ptx::mbar_init(&S.lin_full, 1);
        ptx::mbar_init(&S.lin_done, 1);
        ptx::mbar_init(&S.k1_full, 1);
        ptx::fence_barrier_init();
        ptx::prefetch_tmap(&tm_q);
        ptx::prefetch_tmap(&tm_k);
        ptx::prefetch_tmap(&tm_v);
    }
    if (warp == 5) ptx::tmem_alloc<256>(&S.tmem_base);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (threadIdx.x == 0) TB_TRACE_X(70, 1);
    const uint32_t tmem = S.tmem_base;
    const uint32_t TM_O = tmem + 128;
    // fused linear branch numL = phi(Q) . KV_sel: phi(Q) (A, 2 x 16 KB swizzled
    // K-halves) in v[0..1], KV_sel^T (B) in v[2] + k[0..1].  Linear-first mode
    // (lf: no row_max / den outputs, complement non-empty) runs it BEFORE the
    // main loop, straight into the O accumulator, which then starts as numL at
    // the reference m_ref = log2(linear_mix) (l starts as den_L): the SLA
    // combine (attention.py:416-421) becomes out = O / l, and the prologue
    // already holds the q row that phi(Q) needs.  The producers start once
    // that MMA has released the rings.  Otherwise the same MMA runs after the
    // last PV into the free S columns (end-of-kernel combine).
    const bool fused = a.lin_kv != nullptr && a.linear_mix != 0.0f;
    const bool lf = fused && !EXACT && count < nkv;
    const bool fused_end = fused && !lf;
    // linear-branch staging: phi(Q) (A, 32 KB) and KV_sel^T (B: 32 KB, Q2: both
    // q-blocks' as one N=256 operand, 64 KB).  Q2 stages over q..x, so in lf
    // mode its Q codes are loaded only once the linear MMA has released them.
    uint8_t *lin_a = Q2 ? S.q : S.v[0];
    uint8_t *lin_b = Q2 ? S.v[1] : S.v[2];
    // early (TB_SLA_EARLY, linear-first, not Q2): phi(Q) in TMEM columns 64..127
    // (S buffer 1, free until QK(1)), KV_sel^T's K-halves in v[0] and k[0..1];
    // block j's K slot is (j + KOFF) % KSTAGES and V slot (j + VOFF) % 3, the
    // staging counting as the first use of k[0], k[1], v[0] (released by the
    // linear MMA's commit), so K(0), V(0), V(1) load at once
    const bool early = TB_SLA_EARLY && !Q2 && lf && KSTAGES >= 3;
    const int KOFF = early ? 2 : 0, VOFF = early ? 1 : 0;
    uint8_t *lin_b1 = early ? S.k[0] : lin_b + 16384;       // second K-half of KV_sel^T (non-Q2)
    if (early) lin_b = S.v[0];

#define SLA_CTRL_REGS() \
    do { if (TB_SLA_REGS && TB_SLA_SETMAXNREG) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" :: "n"(CTRL_REGS)); } while (0)
    if (warp == 4) {
        SLA_CTRL_REGS();
        // ---------------------------------------------------- TMA producer (K)
        // the whole warp walks the loop (warp-uniform values, no waterfall
        // loops around the uniform-operand TMA instructions); one lane issues.
        // K and V have their own producer warps, so a K slot freed by QK(j-3)
        // is refilled at once instead of queueing behind the wait for the V
        // slot that PV(j-4) frees.
        const int row0a = (int)(((int64_t)h * nq + qb0) * a.lin_dx);
        const int row0b = (int)(((int64_t)h * nq + qb1) * a.lin_dx);
        // KV_sel^T boxes (64 channels x 128 rows each): Q2 stacks q-block 2n+1's
        // rows under 2n's in each K-half (one N=256 B operand, 32 KB per K-half)
        auto load_lin = [&]() {
            if constexpr (Q2) {
                ptx::mbar_arrive_expect_tx(&S.lin_full, 4 * 16384);
                ptx::tma_load_2d(lin_b, &tm_kv, 0, row0a, &S.lin_full);
                ptx::tma_load_2d(lin_b + 16384, &tm_kv, 0, row0b, &S.lin_full);
                ptx::tma_load_2d(lin_b + 32768, &tm_kv, 64, row0a, &S.lin_full);
                ptx::tma_load_2d(lin_b + 49152, &tm_kv, 64, row0b, &S.lin_full);
            } else {
                ptx::mbar_arrive_expect_tx(&S.lin_full, 2 * 16384);
                ptx::tma_load_2d(lin_b, &tm_kv, 0, row0a, &S.lin_full);
                ptx::tma_load_2d(lin_b1, &tm_kv, 64, row0a, &S.lin_full);
            }
        };
        const bool q_late = Q2 && lf;                   // Q codes after the linear MMA (shared staging)
        if (ptx::elect_one()) {
            if (!q_late) {
                ptx::mbar_arrive_expect_tx(&S.q_full, Q_BYTES);
                ptx::tma_load_3d(S.q, &tm_q, 0, n * BM, h, &S.q_full);
            }
            if (fused) {      // den row of KV_sel: 256 B per q-block
                const __nv_bfloat16 *kvb = reinterpret_cast<const __nv_bfloat16 *>(a.lin_kv);
                ptx::mbar_arrive_expect_tx(&S.k1_full, (Q2 ? 2 : 1) * D * 2);
                ptx::bulk_g2s(S.k1[0], kvb + ((int64_t)row0a + D) * D, D * 2, &S.k1_full);
                if (Q2) ptx::bulk_g2s(S.k1[Q2 ? 1 : 0], kvb + ((int64_t)row0b + D) * D, D * 2, &S.k1_full);
            }
            if (lf) load_lin();
        }
        __syncwarp();
        if (lf && !early) ptx::mbar_wait_sleep(&S.lin_done, 0);   // the linear MMA has released the rings
        if (q_late) {
            if (ptx::elect_one()) {
                ptx::mbar_arrive_expect_tx(&S.q_full, Q_BYTES);
                ptx::tma_load_3d(S.q, &tm_q, 0, n * BM, h, &S.q_full);
            }
            __syncwarp();
        }
        for (int j = 0; j < nsel; j++) {
            const int b = __ldg(sel + j) & 0x0FFFFFFF;
            const int jv = j + KOFF, ks = jv % KSTAGES;
            ptx::mbar_wait_sleep(&S.k_empty[ks], (uint32_t)(((jv / KSTAGES) & 1) ^ 1));
            if (lane == 0) TB_TRACE(j, 10);
            if (ptx::elect_one()) {
#ifdef TB_X_NOLOAD
                ptx::mbar_arrive(&S.k_full[ks]);
#else
                ptx::mbar_arrive_expect_tx(&S.k_full[ks], K_BYTES);
                ptx::tma_load_3d(S.k[ks], &tm_k, 0, b * BN, h, &S.k_full[ks]);
#endif
            }
            __syncwarp();
        }
        if (fused_end) {
            ptx::mbar_wait_sleep(&S.o_final, 0);        // every MMA reading the rings is done
            if (ptx::elect_one()) load_lin();
            __syncwarp();
        }
    } else if (warp == 6) {
        SLA_CTRL_REGS();
        // ---------------------------------------------------- TMA producer (V)
        if (lf && !early) ptx::mbar_wait_sleep(&S.lin_done, 0);
        for (int j = 0; j < nsel; j++) {
            const int b = __ldg(sel + j) & 0x0FFFFFFF;
            const int jv = j + VOFF, vs = jv % VSTAGES;
            ptx::mbar_wait_sleep(&S.v_empty[vs], (uint32_t)(((jv / VSTAGES) & 1) ^ 1));
            if (lane == 0) TB_TRACE(j, 11);
            if (ptx::elect_one()) {
#ifdef TB_X_NOLOAD
                ptx::mbar_arrive(&S.v_full[vs]);
#else
                if constexpr (F8) {       // one 128-channel x 64-token e4m3 box
                    ptx::mbar_arrive_expect_tx(&S.v_full[vs], V_BYTES / 2);
                    ptx::tma_load_3d(S.v[vs], &tm_v, 0, b * BN, h, &S.v_full[vs]);
                } else {
                    ptx::mbar_arrive_expect_tx(&S.v_full[vs], V_BYTES);
                    ptx::tma_load_3d(S.v[vs], &tm_v, 0, b * BN, h, &S.v_full[vs]);
                    ptx::tma_load_3d(S.v[vs] + V_BYTES / 2, &tm_v, 64, b * BN, h, &S.v_full[vs]);
                }
#endif
            }
            __syncwarp();
        }
    } else if (warp == 5) {
        SLA_CTRL_REGS();
        // ------------------------------------------------------- MMA issuer
        // whole warp in the loop, one elected lane issues each MMA group
        constexpr uint32_t ID_QK = ptx::idesc_i8(BM, BN);
        constexpr uint32_t ID_PV = ptx::idesc_bf16(BM, D);
        constexpr uint32_t ID_PV_MN = ptx::idesc_bf16(BM, D) | (1u << 16);   // B = V tile, MN-major
        constexpr uint32_t ID_BIAS = ptx::idesc_bf16(BM, BN);
        constexpr uint32_t ID_PV8_MN = ptx::idesc_e4m3(BM, D) | (1u << 16);  // e4m3 P (TMEM) x V codes, MN-major
        const uint64_t qd = ptx::sdesc_sw128(ptx::smem_u32(S.q));
        // no-swizzle K-major 8x16 bf16 tiles; SBO = 0 makes every 8-row group alias the same rows
        const uint64_t bias_a = ptx::sdesc_noswz_alias(ptx::smem_u32(S.bias_a));
        const uint64_t bias_b = ptx::sdesc_noswz_alias(ptx::smem_u32(S.bias_b));
        // numL = phi(Q) . KV_sel (bf16, K = 128).  B rows: KV_sel^T of one q-block
        // (N = 128, K-half stride 16 KB), or Q2 both stacked (N = 256, K-half
        // stride 32 KB; brow = 128 selects q-block 2n+1's rows alone)
        auto lin_mma = [&](uint32_t dst, int nn, int brow, uint64_t *done) {
            const uint32_t id = ptx::idesc_bf16(BM, nn);
            if (ptx::elect_one()) {
#pragma unroll
                for (int ks = 0; ks < D / 16; ks++) {
                    const int sub = ks >> 2, w = ks & 3;
                    uint8_t *bh = Q2 ? lin_b + sub * 32768 : (sub ? lin_b1 : lin_b);
                    const uint64_t bd = ptx::sdesc_sw128(ptx::smem_u32(bh + brow * 128)) + 2 * w;
                    if (early) {          // A = phi(Q) in TMEM columns 64.. (8 per K16 step)
                        ptx::mma_f16_ts(dst, tmem + 64 + 8 * ks, bd, id, ks > 0 ? 1u : 0u);
                    } else {
                        const uint64_t ad = ptx::sdesc_sw128(ptx::smem_u32(lin_a + sub * 16384)) + 2 * w;
                        ptx::mma_f16(dst, ad, bd, id, ks > 0 ? 1u : 0u);
                    }
                }
                ptx::mma_commit(done);
                if (early) {              // the staging slots of the rings are free again
                    ptx::mma_commit(&S.k_empty[0]);
                    ptx::mma_commit(&S.k_empty[1]);
                    ptx::mma_commit(&S.v_empty[0]);
                }
            }
            __syncwarp();
        };
        auto lin_wait = [&]() {
            MMA_WAIT(&S.phiq_full, 0);
            MMA_WAIT(&S.lin_full, 0);
            ptx::tc_fence_after();
        };
        if (lf && !early) {
            lin_wait();
            if constexpr (Q2) {
                // one N=256 MMA: cols 0-127 = phi(Q) . KV_sel[2n], cols 128-255 (= O) =
                // phi(Q) . KV_sel[2n+1]; warps 0-1 then move their rows' first half into
                // O (lin_fix) before QK(0) may overwrite columns 0-63
                lin_mma(tmem, 2 * D, 0, &S.lin_done);
                MMA_WAIT(&S.lin_fix, 0);
                ptx::tc_fence_after();
            } else {
                lin_mma(TM_O, D, 0, &S.lin_done);       // O starts as numL
            }
        }
        MMA_WAIT(&S.q_full, 0);
        auto pv = [&](int i) {
            const int pb = i & 1, iv = i + VOFF, vs = iv % VSTAGES;
            if (lane == 0) TB_TRACE(i, 13);
            // v_full completes once per real load: the staging use of slots < VOFF has none
            MMA_WAIT(&S.v_full[vs], (uint32_t)((iv / VSTAGES - (vs < VOFF ? 1 : 0)) & 1));
            if (lane == 0) TB_TRACE(i, 14);
            MMA_WAIT(&S.p_full[pb], (uint32_t)((i >> 1) & 1));
            ptx::tc_fence_after();
            if (lane == 0) TB_TRACE(i, 9);
            // V [tokens][channels]: channel-contiguous = MN-major B; atoms 64 ch x 8 tokens
            const uint64_t vd = ptx::sdesc_sw128_mn(ptx::smem_u32(S.v[vs]), V_BYTES / 2, 1024);
            if (ptx::elect_one()) {
#ifndef TB_X_PVN
#define TB_X_PVN (BN / 16)
#endif
                if constexpr (F8) {
                    // e4m3 atoms are 128 channels (128 B) x 8 tokens: K=32 per MMA =
                    // 8 TMEM cols of P (4 per col), 32 token rows of V (4 KB)
                    const uint64_t vd8 = ptx::sdesc_sw128_mn(ptx::smem_u32(S.v[vs]), V_BYTES / 2, 1024);
#pragma unroll
                    for (int k = 0; k < BN / 32; k++)
                        ptx::mma_f8_ts(TM_O, tmem + pb * BN + 8 * k, vd8 + 256 * k, ID_PV8_MN,
                                       (lf || i > 0 || k > 0) ? 1u : 0u);
                } else {
#pragma unroll
                for (int k = 0; k < TB_X_PVN; k++)  // K=16 bf16 per MMA: 8 TMEM cols of P, 16 token rows of V
                    ptx::mma_f16_ts(TM_O, tmem + pb * BN + 8 * k, vd + 128 * k, ID_PV_MN, (lf || i > 0 || k > 0) ? 1u : 0u);
                }
                ptx::mma_commit(&S.pv_done[pb]);
                ptx::mma_commit(&S.v_empty[vs]);
            }
            __syncwarp();
        };
        auto qk = [&](int j) {
            const int jv = j + KOFF, ks = jv % KSTAGES, sb = j & 1;
            if (lane == 0) TB_TRACE(j, 15);
            MMA_WAIT(&S.k_full[ks], (uint32_t)((jv / KSTAGES - (ks < KOFF ? 1 : 0)) & 1));
            ptx::tc_fence_after();
            if (lane == 0) TB_TRACE(j, 8);
            const uint64_t kd = ptx::sdesc_sw128(ptx::smem_u32(S.k[ks]));
            // S_sb last held P_{j-2}, read by PV(j-2), issued earlier: in-order tensor pipe
            if (ptx::elect_one()) {
                // D = 1 x 6291456 + 1 x 6291456 = 1.5*2^23 (bf16 operands, f32 bits) in every cell
                if (TB_SLA_BIAS) ptx::mma_f16(tmem + sb * BN, bias_a, bias_b, ID_BIAS, 0u);
#ifndef TB_X_QKN
#define TB_X_QKN (D / 32)
#endif
#pragma unroll
                for (int k = 0; k < TB_X_QKN; k++)  // K=32 int8 = 32 B per MMA
                    ptx::mma_i8(tmem + sb * BN, qd + 2 * k, kd + 2 * k, ID_QK, (TB_SLA_BIAS || k > 0) ? 1u : 0u);
                ptx::mma_commit(&S.s_full[sb]);
                ptx::mma_commit(&S.k_empty[ks]);
            }
            __syncwarp();
        };
        // QK(j+1) is queued before PV(j) waits for softmax(j): the tensor
        // pipe computes the next scores while the softmax warps work
        if (nsel > 0) qk(0);
        if (early) {                                    // under QK(0); before QK(1) reuses columns 64..
            lin_wait();
            lin_mma(TM_O, D, 0, &S.lin_done);           // O starts as numL
        }
        for (int j = 0; j < nsel; j++) {
            if (j + 1 < nsel) qk(j + 1);
            pv(j);
        }
        if (ptx::elect_one()) ptx::mma_commit(&S.o_final);
        __syncwarp();
        if (fused_end) {                               // into the free S/P columns 0..127
            lin_wait();
            lin_mma(tmem, D, 0, &S.lin_done);
            if constexpr (Q2) {
                // q-block 2n+1's numerator once warps 0-1 have read 2n's (lin_fix)
                MMA_WAIT(&S.lin_fix, 0);
                ptx::tc_fence_after();
                lin_mma(tmem, D, 128, &S.lin_done2);
            }
        }
    } else if (warp == 7) {
        SLA_CTRL_REGS();                            // idle: completes the control warpgroup
    } else {
        if (TB_SLA_REGS && TB_SLA_SETMAXNREG) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" :: "n"(SOFTMAX_REGS));
        // ------------------------------------------------ softmax + epilogue
        const int r = warp * 32 + lane;             // row in tile == TMEM lane
        const int qh = Q2 ? (warp >> 1) : 0;        // Q2: q-block 2n + qh (warp-uniform)
        const int row = n * BM + r;                 // token index
        const bool row_ok = row < L;
        // this warp's TMEM lane quarter, through a shuffle so it is provably
        // warp-uniform: the tcgen05.ld/st addresses below stay in uniform registers
        // (no R2UR per tcgen05 op in the block loop)
#if TB_SLA_UNI
        const uint32_t tw = __shfl_sync(0xffffffffu, tmem + ((uint32_t)(warp * 32) << 16), 0);
        const uint32_t lane_base = 0;
#define TMW tw
#else
        const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
#define TMW tmem
#endif
        const uint32_t tw_o = TMW + (TM_O - tmem);
        const float scale2 = a.scale * LOG2E;
        // F8: V codes carry the per-head scale sv (O accumulates p * v / sv)
        const float vsc = F8 ? __ldg(a.v_scales + h) : 1.0f;
        const float ivsc = F8 ? 1.0f / (vsc == 0.0f ? 1.0f : vsc) : 1.0f;
        // phi(q_row) -> bf16 A operand of the linear MMA (128B-swizzled K halves
        // in lin_a); returns den_L = phi(q) . sum phi(K_b) over the complement.
        // wq: the row already in registers (bf16), else it is (re)loaded.
        const T *qrow = reinterpret_cast<const T *>(a.q) + ((int64_t)h * L + (row_ok ? row : 0)) * D;
        auto stage_phi = [&](const uint4 *wq) {
            if (threadIdx.x == 0) TB_TRACE_X(70, 2);
            ptx::mbar_wait_sleep(&S.k1_full, 0);
            if (threadIdx.x == 0) TB_TRACE_X(70, 3);
            const __nv_bfloat16 *k1 = S.k1[qh];
            float dl = 0.0f;
#pragma unroll
            for (int kc = 0; kc < D / 8; kc++) {
                uint32_t pk[4];
                float xq[8];
                if (sizeof(T) == 2 && wq != nullptr) {
                    const __nv_bfloat162 *b2 = reinterpret_cast<const __nv_bfloat162 *>(&wq[kc]);
#pragma unroll
                    for (int i = 0; i < 4; i++) { const float2 f = __bfloat1622float2(b2[i]); xq[2 * i] = f.x; xq[2 * i + 1] = f.y; }
                } else {
                    load8(qrow + kc * 8, xq);
                    if (!row_ok) {
#pragma unroll
                        for (int i = 0; i < 8; i++) xq[i] = 0.0f;
                    }
                }
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    // branch-free phi (attention.py:287-290); padding rows read
                    // q = 0 and are never stored
                    const float x0 = xq[2 * u], x1 = xq[2 * u + 1];
                    const float f0 = x0 >= 0.0f ? x0 + 1.0f : ex2(x0 * LOG2E);
                    const float f1 = x1 >= 0.0f ? x1 + 1.0f : ex2(x1 * LOG2E);
                    dl = fmaf(f0, __bfloat162float(k1[kc * 8 + 2 * u]), dl);
                    dl = fmaf(f1, __bfloat162float(k1[kc * 8 + 2 * u + 1]), dl);
                    __nv_bfloat162 pp = __floats2bfloat162_rn(f0, f1);
                    pk[u] = *reinterpret_cast<uint32_t *>(&pp);
                }
                uint8_t *dst = lin_a + (kc >> 3) * 16384 + r * 128 + (((kc & 7) ^ (r & 7)) * 16);
                *reinterpret_cast<uint4 *>(dst) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
            }
            if (threadIdx.x == 0) TB_TRACE_X(70, 4);
            ptx::fence_async_smem();
            ptx::mbar_arrive(&S.phiq_full);
            if (threadIdx.x == 0) TB_TRACE_X(70, 5);
            return dl;
        };
        float corr_e = 0.0f, den_e = 0.0f;             // early: this row's q . k_mean and den_L
        if (early) {
            // Prologue per row (thread = row = TMEM lane): corr = q . k_mean,
            // phi(q) -> bf16 pairs -> TMEM columns 64..127 (the linear MMA's A
            // operand), den_L = phi(q) . sum phi(K_b) over the complement.
            const float *kmh = a.k_mean + (int64_t)h * D;
            // bf16: the whole row (16 x 16 B) in flight before the den-row wait
            uint4 qv[sizeof(T) == 2 ? 16 : 1];
            if constexpr (sizeof(T) == 2) {
#pragma unroll
                for (int i = 0; i < 16; i++)
                    qv[i] = row_ok ? __ldg(reinterpret_cast<const uint4 *>(qrow) + i) : make_uint4(0, 0, 0, 0);
            }
            ptx::mbar_wait_sleep(&S.k1_full, 0);
            const __nv_bfloat16 *k1 = S.k1[0];
#pragma unroll
            for (int c32 = 0; c32 < D; c32 += 32) {
                uint32_t pk[16];
#pragma unroll
                for (int c8 = 0; c8 < 32; c8 += 8) {
                    float x[8];
                    if constexpr (sizeof(T) == 2) {
                        const __nv_bfloat162 *b2 = reinterpret_cast<const __nv_bfloat162 *>(&qv[(c32 + c8) >> 3]);
#pragma unroll
                        for (int i = 0; i < 4; i++) { const float2 f = __bfloat1622float2(b2[i]); x[2 * i] = f.x; x[2 * i + 1] = f.y; }
                    } else if (row_ok) {
                        load8(qrow + c32 + c8, x);
                    } else {
#pragma unroll
                        for (int i = 0; i < 8; i++) x[i] = 0.0f;
                    }
                    const float4 ka = __ldg(reinterpret_cast<const float4 *>(kmh + c32 + c8));
                    const float4 kb = __ldg(reinterpret_cast<const float4 *>(kmh + c32 + c8 + 4));
                    const float km8[8] = {ka.x, ka.y, ka.z, ka.w, kb.x, kb.y, kb.z, kb.w};
                    const uint4 kw = *reinterpret_cast<const uint4 *>(k1 + c32 + c8);
                    const __nv_bfloat162 *k2 = reinterpret_cast<const __nv_bfloat162 *>(&kw);
#pragma unroll
                    for (int u = 0; u < 4; u++) {
                        const float x0 = x[2 * u], x1 = x[2 * u + 1];
                        corr_e = fmaf(x0, km8[2 * u], corr_e);
                        corr_e = fmaf(x1, km8[2 * u + 1], corr_e);
                        const float f0 = x0 >= 0.0f ? x0 + 1.0f : ex2(x0 * LOG2E);
                        const float f1 = x1 >= 0.0f ? x1 + 1.0f : ex2(x1 * LOG2E);
                        const float2 kk = __bfloat1622float2(k2[u]);
                        den_e = fmaf(f0, kk.x, fmaf(f1, kk.y, den_e));
                        __nv_bfloat162 pp = F8 ? __floats2bfloat162_rn(f0 * ivsc, f1 * ivsc) : __floats2bfloat162_rn(f0, f1);
                        pk[(c8 >> 1) + u] = *reinterpret_cast<uint32_t *>(&pp);
                    }
                }
                ptx::tmem_st16(TMW + lane_base + 64 + (c32 >> 1), pk);
            }
            ptx::tmem_wait_st();
            ptx::tc_fence_before();
            ptx::mbar_arrive(&S.phiq_full);
        } else
        // Prologue, warp-cooperative and coalesced: each warp walks its 32 rows
        // two at a time (lanes 0-15 row 2i, 16-31 row 2i+1, 16 B of the row per
        // lane), so every load instruction reads 512 contiguous bytes.  Per row:
        // corr = q . k_mean (unquantized q, f32; a tolerance-level quantity whose
        // reference order is an sgemm's) and, in lf mode, phi(q) -> the bf16 A
        // operand of the linear MMA (128B-swizzled K halves in lin_a) and
        // den_L = phi(q) . sum phi(K_b) over the complement; 16-lane shuffle
        // reductions, results through smem (read after the barrier below).
        {
            const int half = lane >> 4, cl = lane & 15;
            float km[8], kk[8];
            {
                const float4 *km4 = reinterpret_cast<const float4 *>(a.k_mean + (int64_t)h * D + cl * 8);
                const float4 ka = __ldg(km4), kb = __ldg(km4 + 1);
                km[0] = ka.x; km[1] = ka.y; km[2] = ka.z; km[3] = ka.w;
                km[4] = kb.x; km[5] = kb.y; km[6] = kb.z; km[7] = kb.w;
            }
            const T *qbase = reinterpret_cast<const T *>(a.q) + (int64_t)h * L * D + cl * 8;
            const int rbase = warp * 32 + half;
            uint4 qv[sizeof(T) == 2 ? 16 : 1];
            if constexpr (sizeof(T) == 2) {
#pragma unroll
                for (int it = 0; it < 16; it++) {
                    const int rowi = n * BM + rbase + 2 * it;
                    qv[it] = rowi < L ? __ldg(reinterpret_cast<const uint4 *>(qbase + (int64_t)rowi * D))
                                      : make_uint4(0, 0, 0, 0);
                }
            }
            if (lf) {
                ptx::mbar_wait_sleep(&S.k1_full, 0);
                const uint4 kw = *reinterpret_cast<const uint4 *>(S.k1[qh] + cl * 8);
                const __nv_bfloat162 *k2 = reinterpret_cast<const __nv_bfloat162 *>(&kw);
#pragma unroll
                for (int i = 0; i < 4; i++) { const float2 f = __bfloat1622float2(k2[i]); kk[2 * i] = f.x; kk[2 * i + 1] = f.y; }
            }
#pragma unroll
            for (int it = 0; it < 16; it++) {
                const int rr = rbase + 2 * it;
                float x[8];
                if constexpr (sizeof(T) == 2) {
                    const __nv_bfloat162 *b2 = reinterpret_cast<const __nv_bfloat162 *>(&qv[it]);
#pragma unroll
                    for (int i = 0; i < 4; i++) { const float2 f = __bfloat1622float2(b2[i]); x[2 * i] = f.x; x[2 * i + 1] = f.y; }
                } else {
                    const int rowi = n * BM + rr;
                    if (rowi < L) {
                        load8(qbase + (int64_t)rowi * D, x);
                    } else {
#pragma unroll
                        for (int i = 0; i < 8; i++) x[i] = 0.0f;
                    }
                }
                float cp = 0.0f, dp = 0.0f;
#pragma unroll
                for (int i = 0; i < 8; i++) cp = fmaf(x[i], km[i], cp);
                if (lf) {
                    uint32_t pk[4];
#pragma unroll
                    for (int u = 0; u < 4; u++) {
                        const float x0 = x[2 * u], x1 = x[2 * u + 1];
                        const float f0 = x0 >= 0.0f ? x0 + 1.0f : ex2(x0 * LOG2E);
                        const float f1 = x1 >= 0.0f ? x1 + 1.0f : ex2(x1 * LOG2E);
                        dp = fmaf(f0, kk[2 * u], fmaf(f1, kk[2 * u + 1], dp));
                        __nv_bfloat162 pp = F8 ? __floats2bfloat162_rn(f0 * ivsc, f1 * ivsc) : __floats2bfloat162_rn(f0, f1);
                        pk[u] = *reinterpret_cast<uint32_t *>(&pp);
                    }
                    uint8_t *dst = lin_a + (cl >> 3) * 16384 + rr * 128 + (((cl & 7) ^ (rr & 7)) * 16);
                    *reinterpret_cast<uint4 *>(dst) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                }
#pragma unroll
                for (int o = 8; o > 0; o >>= 1) {
                    cp += __shfl_xor_sync(0xffffffffu, cp, o);
                    dp += __shfl_xor_sync(0xffffffffu, dp, o);
                }
                if (cl == 0) { S.corr_s[rr] = cp; S.den_s[rr] = dp; }
            }
            if (lf) {
                ptx::fence_async_smem();
                ptx::mbar_arrive(&S.phiq_full);
            }
        }
        if (threadIdx.x == 0) TB_TRACE_X(70, 6);
        const float sq0 = __ldg(a.q_scales + (int64_t)h * nq + qb0);
        const float sq1 = Q2 ? __ldg(a.q_scales + (int64_t)h * nq + qb1) : sq0;
        const float *ksc = a.k_scales + (int64_t)h * nkv;
        const int last_blk = nkv - 1;
        const int last_ext = L - last_blk * BN;
        // m_ref: the running reference (log2 units) the exponentials are taken
        // against.  Fast path (EXACT == false): no per-block row max at all --
        // p = 2^(logit2 - m_ref) is computed straight away and the block is
        // accepted when its row sum stays <= 2^60 (finite, far from f32 / bf16
        // overflow); otherwise (first block: m_ref = -inf gives inf / NaN) the
        // warp takes the exact path below: row max, lazy O rebase when the max
        // outgrows m_ref by > 8, recompute.  The softmax and the SLA combine
        // are invariant to the reference (attention.py:416-421: num and den
        // carry the same exp(-ref)), so only rounding differs.  EXACT == true
        // (row_max / den outputs requested) runs the exact path every block
        // and reports the true row max like _sparse_branch (attention.py:385-389).
        // per selected block: logit slope and ragged flag (smem, read once per block)
        for (int j = r; j < nsel; j += BM) {
            const int e = __ldg(sel + j);
            const int b = e & 0x0FFFFFFF;
            const float skb = __ldg(ksc + b);
            S.c1[j] = Q2 ? skb * scale2 : sq0 * skb * scale2;   // Q2: the q-half's sq is applied per warp
            S.rag[j] = (uint8_t)((((b == last_blk) && last_ext < BN) ? 4 : 0) | (Q2 ? (e >> 28) & 3 : 3));
        }
        if (threadIdx.x == 0) TB_TRACE_X(70, 7);
        ptx::named_bar_sync(1, BM);
        if (Q2 && lf && qh == 0) {
            // the N=256 linear MMA left q-block 2n's numerator in columns 0-127:
            // rows 0-63 move it into O (2n+1's is already there), then QK(0) may
            // overwrite those columns
            ptx::mbar_wait_sleep(&S.lin_done, 0);
            ptx::tc_fence_after();
#pragma unroll 1
            for (int c = 0; c < D; c += 16) {
                uint32_t o[16];
                ptx::tmem_ld16(TMW + lane_base + c, o);
                ptx::tmem_wait_ld();
                ptx::tmem_st16(tw_o + lane_base + c, o);
            }
            ptx::tmem_wait_st();
            ptx::tc_fence_before();
            ptx::mbar_arrive(&S.lin_fix);
        }
        TB_PH(ph_t1 = clock64());
        if (threadIdx.x == 0) TB_TRACE_X(70, 8);
        const float c0 = (row_ok ? (early ? corr_e : S.corr_s[r]) : 0.0f) * scale2;
        const float den_l = early ? den_e : S.den_s[r];
        // lf: O already holds numL at the reference log2(linear_mix), l = den_L.
        // (Warp-uniform start: the rebase below is warp-collective.  A row with
        // l == 0 -- phi(q) underflowed, or a padding row -- whose exponentials
        // all underflow is caught by the l + psum > 0 test and rebased down.)
        float m_ref = lf ? __log2f(a.linear_mix) : -INFINITY, m_true = -INFINITY;
        float l = lf ? den_l : 0.0f;
        for (int j = 0; j < nsel; j++) {
            const int sb = j & 1;
            const uint32_t flags = S.rag[j];
            if (Q2 && !((flags >> qh) & 1u)) {
                // block selected only by the other q-block of the tile: P = 0 for these
                // rows (stored once QK(j) has written S_j, which P_j overwrites)
                SM_WAIT(&S.s_full[sb], (uint32_t)((j >> 1) & 1));
                ptx::tc_fence_after();
                uint32_t z[16];
#pragma unroll
                for (int i = 0; i < 16; i++) z[i] = 0u;
                ptx::tmem_st16(TMW + lane_base + sb * BN, z);
                if (!F8) ptx::tmem_st16(TMW + lane_base + sb * BN + 16, z);
                ptx::tmem_wait_st();
                ptx::tc_fence_before();
                ptx::mbar_arrive(&S.p_full[sb]);
                continue;
            }
            const float c1 = Q2 ? (qh ? sq1 : sq0) * S.c1[j] : S.c1[j];
            // s32 scores as the floats M + s (M = 1.5*2^23, exact): fold -M*c1 into the offset
            const float c0m = fmaf(-12582912.0f, c1, c0);
            if (threadIdx.x == 0) TB_TRACE(j, 0);
            SM_WAIT(&S.s_full[sb], (uint32_t)((j >> 1) & 1));
            ptx::tc_fence_after();
            if (threadIdx.x == 0) TB_TRACE(j, 1);
            uint32_t s[4][16];
            auto load_s = [&]() {
#pragma unroll
                for (int q4 = 0; q4 < 4; q4++) ptx::tmem_ld16(TMW + lane_base + sb * BN + q4 * 16, s[q4]);
                ptx::tmem_wait_ld();
            };
            load_s();
            if (threadIdx.x == 0) TB_TRACE(j, 4);
            const bool ragged = (flags & 4u) != 0;                    // uniform per CTA
            const int lim = ragged ? last_ext : BN;
            // scores as floats M + s (exact, |s| < 2^22), monotone in s
            auto xm = [&](int i) {
                return __int_as_float((int)s[i >> 4][i & 15] + (TB_SLA_BIAS ? 0 : 0x4B400000));
            };
            float2 psum2[4];
            uint32_t pk[2][16];
            // P from the registers s[] (consumed as it goes, so the exact path
            // below reloads S from TMEM instead of keeping 64 values alive)
            auto make_p = [&](auto rg, float off) {
                constexpr bool RG = decltype(rg)::value;
                const float2 c12 = make_float2(c1, c1), off2 = make_float2(off, off);
                const float2 cu = make_float2(c1 * 0.00390625f, c1 * 0.00390625f);
                const float ou = fmaf(off, 0.00390625f, 0.48828125f);        // off/256 + 125/256
                const float2 ou2 = make_float2(ou, ou);
#pragma unroll
                for (int u = 0; u < 4; u++) psum2[u] = make_float2(0.0f, 0.0f);
#pragma unroll
                for (int i = 0; i < 64; i += 2) {
                    // 3 of every 8 pairs (3/8 of the exponentials) on the FMA pipe, the rest on MUFU
                    constexpr int PP = TB_SLA_PP;                   // pair-slot mask {1, 4, 6} of 8
                    float p0, p1;
                    if ((PP >> ((i >> 1) & 7)) & 1) {
                        const float2 e = ex2_poly2_sat(ptx::ffma2_sat(make_float2(xm(i), xm(i + 1)), cu, ou2));
                        p0 = e.x;
                        p1 = e.y;
                    } else {
                        const float2 y = ptx::ffma2(make_float2(xm(i), xm(i + 1)), c12, off2);   // FFMA2
                        p0 = ex2(y.x);
                        p1 = ex2(y.y);
                    }
                    if (RG) {
                        if (i >= lim) p0 = 0.0f;
                        if (i + 1 >= lim) p1 = 0.0f;
                    }
#ifdef TB_X_NOSUM
                    if (i == 0) psum2[0] = make_float2(p0, p1);
#else
                    psum2[(i >> 1) & 3] = ptx::fadd2(psum2[(i >> 1) & 3], make_float2(p0, p1));
#endif
                    if constexpr (F8) {      // four e4m3 per TMEM column (K order = byte order)
                        const uint32_t h2 = __nv_cvt_float2_to_fp8x2(make_float2(p0, p1), __NV_SATFINITE, __NV_E4M3);
                        if ((i & 2) == 0) pk[0][i >> 2] = h2;
                        else pk[0][i >> 2] |= h2 << 16;
                    } else {
                    __nv_bfloat162 pp = __floats2bfloat162_rn(p0, p1);
                    pk[i >> 5][(i >> 1) & 15] = *reinterpret_cast<uint32_t *>(&pp);
                    }
                }
                const float2 ps = ptx::fadd2(ptx::fadd2(psum2[0], psum2[1]), ptx::fadd2(psum2[2], psum2[3]));
                return ps.x + ps.y;
            };
            auto run_p = [&](float off) {
                return ragged ? make_p(std::integral_constant<bool, true>(), off)
                              : make_p(std::integral_constant<bool, false>(), off);
            };
            float psum = 0.0f;
            bool slow = EXACT;
            if (!EXACT) {
                psum = run_p(c0m - m_ref);
                // F8: every p <= 448 (e4m3 max) follows from a row sum <= 448
                slow = __any_sync(0xffffffffu, !(psum <= (F8 ? 448.0f : 0x1p60f)) || !(l + psum > 0.0f));
            }
            if (slow) {
                if (!EXACT) load_s();         // S is intact in TMEM until P is stored
                // exact row max of the block: logit2 is affine in the exact s32
                // score with slope c1 (uniform sign per CTA) -> max/min of M + s
                float sx;
                if (!ragged) {
                    // 4 independent 3-input max/min chains (depth 8 instead of 31)
                    float a4[4];
                    if (c1 >= 0.0f) {
#pragma unroll
                        for (int u = 0; u < 4; u++) a4[u] = xm(u);
#pragma unroll
                        for (int i = 4; i < 64; i += 8)
#pragma unroll
                            for (int u = 0; u < 4; u++) a4[u] = fmaxf(a4[u], fmaxf(xm(i + 2 * u), xm(i + 2 * u + 1)));
                        sx = fmaxf(fmaxf(a4[0], a4[1]), fmaxf(a4[2], a4[3]));
                    } else {
#pragma unroll
                        for (int u = 0; u < 4; u++) a4[u] = xm(u);
#pragma unroll
                        for (int i = 4; i < 64; i += 8)
#pragma unroll
                            for (int u = 0; u < 4; u++) a4[u] = fminf(a4[u], fminf(xm(i + 2 * u), xm(i + 2 * u + 1)));
                        sx = fminf(fminf(a4[0], a4[1]), fminf(a4[2], a4[3]));
                    }
                } else {
                    sx = xm(0);
#pragma unroll
                    for (int i = 1; i < 64; i++)      // static indices keep s[] in registers
                        if (i < lim) sx = (c1 >= 0.0f) ? fmaxf(sx, xm(i)) : fminf(sx, xm(i));
                }
                const float mx = fmaf(sx, c1, c0m);
                if (threadIdx.x == 0) TB_TRACE(j, 2);
                m_true = fmaxf(m_true, mx);
                if (m_ref == -INFINITY) {
                    m_ref = mx;                       // first block of the row: nothing accumulated yet
                } else {
                    // lazy rebase of O when a row's max outgrows its reference by
                    // > 8 (p <= 256).  tcgen05.ld/st are warp-collective, so the
                    // decision is made per warp; rows that do not need it use 1.
                    const bool need = mx > m_ref + 8.0f || (l == 0.0f && mx < m_ref - 8.0f);
                    if (__any_sync(0xffffffffu, need)) {
                        if (j > 0) ptx::mbar_wait_sleep(&S.pv_done[(j - 1) & 1], (uint32_t)(((j - 1) >> 1) & 1));
                        else ptx::mbar_wait_sleep(&S.lin_done, 0);   // lf: O = numL
                        ptx::tc_fence_after();
                        const float alpha = need ? (l == 0.0f ? 0.0f : ex2(m_ref - mx)) : 1.0f;   // l == 0: O == 0
#pragma unroll 1
                        for (int c = 0; c < D; c += 16) {
                            uint32_t o[16];
                            ptx::tmem_ld16(tw_o + lane_base + c, o);
                            ptx::tmem_wait_ld();
#pragma unroll
                            for (int i = 0; i < 16; i++) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
                            ptx::tmem_st16(tw_o + lane_base + c, o);
                        }
                        l *= alpha;
                        if (need) m_ref = mx;
                    }
                }
                psum = run_p(c0m - m_ref);
            }
            if (threadIdx.x == 0) TB_TRACE(j, 5);
            l += psum;
            // P_j overwrites S_j's first 32 columns (A operand of PV, bf16x2 per column)
            ptx::tmem_st16(TMW + lane_base + sb * BN, pk[0]);
            if (!F8) ptx::tmem_st16(TMW + lane_base + sb * BN + 16, pk[1]);
            ptx::tmem_wait_st();
            if (threadIdx.x == 0) TB_TRACE(j, 6);
            ptx::tc_fence_before();
            ptx::mbar_arrive(&S.p_full[sb]);
            if (threadIdx.x == 0) TB_TRACE(j, 3);
            if (threadIdx.x == 96) TB_TRACE(j, 12);
        }
        TB_PH(ph_t2 = clock64());
        if (!EXACT) m_true = m_ref;                  // combine against the reference (exact in math)
        // ------------------------------------------------------- epilogue
        if (threadIdx.x == 0) TB_TRACE_X(71, 0);
        ptx::mbar_wait_sleep(&S.o_final, 0);
        ptx::tc_fence_after();
        if (threadIdx.x == 0) TB_TRACE_X(71, 1);
        float den_fused = 0.0f;
        if (fused_end) {
            den_fused = stage_phi(nullptr);
            if (threadIdx.x == 0) TB_TRACE_X(71, 2);
            // Q2: rows 64-127 read q-block 2n+1's numerator, written into the same
            // columns after rows 0-63 are done with 2n's (lin_fix below)
            ptx::mbar_wait_sleep((Q2 && qh == 1) ? &S.lin_done2 : &S.lin_done, 0);
            ptx::tc_fence_after();
            if (threadIdx.x == 0) TB_TRACE_X(71, 3);
        }
        // rebase to the true row max (natural-log units for the combine)
        const float f = ex2(m_ref - m_true);
        const float m_nat = m_true * LN2;           // log2-domain max -> natural units
        const float l_true = l * f;
        const bool lin = fused_end || (!lf && a.num_l != nullptr && a.linear_mix != 0.0f);
        const int64_t lin_ld = a.lin_ld ? a.lin_ld : D;
        const int64_t lin_hs = a.lin_hs ? a.lin_hs : (int64_t)L * lin_ld;
        const float *nl_row = (lin && !fused_end) ? a.num_l + (int64_t)h * lin_hs + (int64_t)row * lin_ld : nullptr;
        const float *dl_ptr = (lin && !fused_end) ? (a.lin_ld ? nl_row + D : a.den_l + (int64_t)h * L + row) : nullptr;
        float ss = f, shrink = 0.0f, den = l_true;
        if (lin && row_ok) {
            const float ref = fmaxf(m_nat, 0.0f);
            const float e_ss = expf(m_nat - ref);
            shrink = expf(-ref) * a.linear_mix;
            den = l_true * e_ss + shrink * (fused_end ? den_fused : *dl_ptr);
            ss = f * e_ss;
        }
        const float inv = 1.0f / den;
        ss *= vsc;                                  // F8: O holds sum p * v / sv
        const float fo = f * vsc;
        if (row_ok) {
            if (a.row_max) a.row_max[(int64_t)h * L + row] = m_nat;
            if (a.den) a.den[(int64_t)h * L + row] = l_true;
        }
        // final values of 16 output channels from TMEM (O, and the end-of-kernel
        // linear numerator when fused_end) and the combine factors above
        auto out16 = [&](int c, float (&v)[16]) {
            uint32_t o[16], nlt[16];
            ptx::tmem_ld16(tw_o + lane_base + c, o);
            if (fused_end) ptx::tmem_ld16(TMW + lane_base + c, nlt);
            ptx::tmem_wait_ld();
            if (fused_end) {
#pragma unroll
                for (int i = 0; i < 16; i++)
                    v[i] = (__uint_as_float(o[i]) * ss + shrink * __uint_as_float(nlt[i])) * inv;
            } else if (lin) {
#pragma unroll
                for (int i = 0; i < 16; i += 4) {
                    const float4 nl = row_ok ? *reinterpret_cast<const float4 *>(nl_row + c + i) : make_float4(0.f, 0.f, 0.f, 0.f);
                    v[i] = (__uint_as_float(o[i]) * ss + shrink * nl.x) * inv;
                    v[i + 1] = (__uint_as_float(o[i + 1]) * ss + shrink * nl.y) * inv;
                    v[i + 2] = (__uint_as_float(o[i + 2]) * ss + shrink * nl.z) * inv;
                    v[i + 3] = (__uint_as_float(o[i + 3]) * ss + shrink * nl.w) * inv;
                }
            } else {
#pragma unroll
                for (int i = 0; i < 16; i++) v[i] = __uint_as_float(o[i]) * fo * inv;
            }
        };
        if (a.out_dtype == TB_I8) {
            // The out-projection's A operand straight from the epilogue: the
            // bf16-rounded tile (what a bf16 output would hold) quantized as one
            // 128 x 128 block -- absmax over the tile's valid rows (4 warps,
            // named barrier), then the codes in a second TMEM pass
            // (quantize_blockwise semantics, blockquant.py:91-110)
            float am = 0.0f;
#pragma unroll 1
            for (int c = 0; c < D; c += 16) {
                float v[16];
                out16(c, v);
#pragma unroll
                for (int i = 0; i < 16; i++) am = fmaxf(am, fabsf(__bfloat162float(__float2bfloat16_rn(v[i]))));
            }
            am = warp_max<32>(row_ok ? am : 0.0f);
            if (lane == 0) S.corr_s[warp] = am;       // the prologue's scratch, long since consumed
            ptx::named_bar_sync(1, BM);
            am = fmaxf(fmaxf(S.corr_s[0], S.corr_s[1]), fmaxf(S.corr_s[2], S.corr_s[3]));
            const float sc = quant_scale(am);
            // destination: this rank's buffers, or (fused Ulysses return) the
            // token owner's buffers in peer memory -- a 128-row tile never
            // straddles two owners (peer_rows % 128 == 0)
            int8_t *obase = reinterpret_cast<int8_t *>(a.out);
            float *sbase = a.out_scales;
            int64_t orow0 = (int64_t)n * BM, ocols = a.H * D, ohead = h;
            if (a.out_peers) {
                const int64_t owner = orow0 / a.peer_rows;
                obase = reinterpret_cast<int8_t *>(a.out_peers[owner]);
                sbase = a.scale_peers[owner];
                orow0 -= owner * a.peer_rows;
                ocols = a.out_heads * D;
                ohead = a.head0 + h;
            }
            if (threadIdx.x == 0) sbase[(orow0 / BM) * (ocols / D) + ohead] = sc;
            const float safe = (sc == 0.0f) ? 1.0f : sc;
            const float rq = __frcp_rn(safe);
            const bool exq = !(safe >= 1.17549435e-38f && rq <= 3.0e38f);   // subnormal scale: exact division
            int8_t *dst = obase + (orow0 + r) * ocols + ohead * D;
#pragma unroll 1
            for (int c = 0; c < D; c += 16) {
                float v[16];
                out16(c, v);
#pragma unroll
                for (int i = 0; i < 16; i++) v[i] = __bfloat162float(__float2bfloat16_rn(v[i]));
                uint32_t w[4];
                quant16_fast(v, safe, rq, exq, w);
                if (row_ok) *reinterpret_cast<uint4 *>(dst + c) = make_uint4(w[0], w[1], w[2], w[3]);
            }
        } else {
#pragma unroll 1
            for (int c = 0; c < D; c += 16) {
                float v[16];
                out16(c, v);
                if (!row_ok) continue;
                const int64_t off = ((int64_t)h * L + row) * D + c;
                if (a.out_dtype == TB_BF16) {
                    __nv_bfloat16 *dst = reinterpret_cast<__nv_bfloat16 *>(a.out) + off;
#pragma unroll
                    for (int i = 0; i < 16; i += 8) {
                        uint4 w;
                        __nv_bfloat162 *p = reinterpret_cast<__nv_bfloat162 *>(&w);
#pragma unroll
                        for (int u = 0; u < 4; u++) p[u] = __floats2bfloat162_rn(v[i + 2 * u], v[i + 2 * u + 1]);
                        *reinterpret_cast<uint4 *>(dst + i) = w;
                    }
                } else {
                    float *dst = a.out + off;
#pragma unroll
                    for (int i = 0; i < 16; i += 4)
                        *reinterpret_cast<float4 *>(dst + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
                }
            }
        }
        if (Q2 && fused_end && qh == 0) {            // done reading columns 0-127: q-block 2n+1's turn
            ptx::tc_fence_before();
            ptx::mbar_arrive(&S.lin_fix);
        }
    }
    if (threadIdx.x == 0) TB_TRACE_X(71, 4);
    TB_PH(if (threadIdx.x == 0) tb_phase_done(ph_t0, ph_g0, ph_t1, ph_t2));
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 5) ptx::tmem_dealloc<256>(tmem);
}
#undef TMW

int sla_simt(const tb_sla_args *a, cudaStream_t st);

bool sla_tc_supported(const tb_sla_args *a) {
    const int64_t nkv = cdiv(a->L, 64);
    // q_block 64: union lists from tb_pair_union, at most max_sel<true>() per tile
    const bool q2 = a->q_block == 64 && a->pair_idx != nullptr && a->pair_cnt != nullptr &&
                    a->pair_ld >= 2 * a->count &&
                    imin64(2 * a->count, nkv) <= sla::max_sel<true>();
    return a->quantized && a->d == 128 && (a->q_block == 128 || q2) && a->kv_block == 64 &&
           (a->dtype == TB_BF16 || a->vt != nullptr) && a->L >= 128 &&
           (a->dtype == TB_BF16 || a->dtype == TB_F32) && a->count >= 1 && a->count <= sla::MAX_SEL &&
           (a->lin_kv == nullptr || a->lin_dx >= a->d + 1);
}

int sla_tc(const tb_sla_args *a, cudaStream_t st) {
    using namespace sla;
    const bool q2 = a->q_block == 64;
    const int64_t nq = cdiv(a->L, a->q_block), nkv = cdiv(a->L, BN);
    CUtensorMap tq, tk, tv;
    bool ok = make_tmap_3d(&tq, a->q_codes, CU_TENSOR_MAP_DATA_TYPE_UINT8, D, a->L, a->H, D, a->L * D, D, BM, 1) &&
              make_tmap_3d(&tk, a->k_codes, CU_TENSOR_MAP_DATA_TYPE_UINT8, D, a->L, a->H, D, a->L * D, D, BN, 1) &&
              (a->v_fp8 ? make_tmap_3d(&tv, a->v_fp8, CU_TENSOR_MAP_DATA_TYPE_UINT8, D, a->L, a->H, D, a->L * D, D, BN, 1)
                        : make_tmap_3d(&tv, a->dtype == TB_BF16 ? a->v : a->vt, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, D,
                                       a->L, a->H, D * 2, a->L * D * 2, 64, BN, 1));
    CUtensorMap tkv = tq;
    if (a->lin_kv)
        ok = ok && make_tmap_2d(&tkv, a->lin_kv, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, D, a->H * nq * a->lin_dx, D * 2,
                                64, 128);
    if (!ok) return fail(TB_ECUDA, "cuTensorMapEncodeTiled failed (sla)");
    // the exact-max variant only when the caller asks for the sparse-branch stats
    const bool exact = a->row_max != nullptr || a->den != nullptr;
    dim3 grid((unsigned)cdiv(a->L, BM), (unsigned)a->H);
    auto launch = [&](auto kern, size_t smem) {
#ifdef TB_SLA_TRACE
        // trace build only: TB_SLA_SMEM_PAD extra bytes (e.g. one CTA per SM, for
        // per-block phase timings without a co-resident CTA)
        if (const char *e = getenv("TB_SLA_SMEM_PAD")) smem += (size_t)atol(e);
#endif
        smem_attr(kern, (int)smem);
        kern<<<grid, THREADS, smem, st>>>(tq, tk, tv, tkv, *a, (int)nq, (int)nkv);
    };
    constexpr size_t S1 = sizeof(SmemT<false>), S2 = sizeof(SmemT<true>);
    if (q2) {
        if (a->v_fp8) {
            if (exact) launch(sla_tc_kernel<__nv_bfloat16, true, true, true>, S2);
            else launch(sla_tc_kernel<__nv_bfloat16, false, true, true>, S2);
        } else if (a->dtype == TB_BF16) {
            if (exact) launch(sla_tc_kernel<__nv_bfloat16, true, false, true>, S2);
            else launch(sla_tc_kernel<__nv_bfloat16, false, false, true>, S2);
        } else {
            if (exact) launch(sla_tc_kernel<float, true, false, true>, S2);
            else launch(sla_tc_kernel<float, false, false, true>, S2);
        }
    } else if (a->v_fp8) {
        if (exact) launch(sla_tc_kernel<__nv_bfloat16, true, true>, S1);
        else launch(sla_tc_kernel<__nv_bfloat16, false, true>, S1);
    } else if (a->dtype == TB_BF16) {
        if (exact) launch(sla_tc_kernel<__nv_bfloat16, true>, S1);
        else launch(sla_tc_kernel<__nv_bfloat16, false>, S1);
    } else {
        if (exact) launch(sla_tc_kernel<float, true>, S1);
        else launch(sla_tc_kernel<float, false>, S1);
    }
    return check_launch("sla_tc");
}

}  // namespace tb

using namespace tb;

extern "C" int tb_sla_attention(const tb_sla_args *a, void *stream) {
    TB_REQUIRE(a != nullptr, "null args");
    TB_REQUIRE(a->H >= 0 && a->L >= 1 && a->d >= 1, "bad shape");
    TB_REQUIRE(a->q_block >= 1 && a->kv_block >= 1, "block sizes must be >= 1");
    TB_REQUIRE(a->q_block <= a->L && a->kv_block <= a->L, "block sizes exceed seq");
    TB_REQUIRE(a->count >= 1 && a->count <= cdiv(a->L, a->kv_block), "bad count");
    TB_REQUIRE(a->dtype == TB_F32 || a->dtype == TB_BF16, "dtype must be f32 or bf16");
    TB_REQUIRE(!a->quantized || (a->q_codes && a->k_codes && a->q_scales && a->k_scales && a->k_mean),
               "quantized branch needs codes, scales and k_mean");
    if (a->H == 0) return TB_OK;
    cudaStream_t st = as_stream(stream);
    TB_REQUIRE(a->out_dtype != TB_I8 || ((a->out_scales != nullptr || a->out_peers != nullptr) && sla_tc_supported(a) &&
                                         a->row_max == nullptr && a->den == nullptr),
               "int8 output needs the tensor-core kernel and out_scales (and no row_max / den)");
    TB_REQUIRE(a->out_peers == nullptr ||
                   (a->out_dtype == TB_I8 && a->scale_peers != nullptr && a->peer_rows > 0 && a->peer_rows % 128 == 0 &&
                    a->head0 >= 0 && a->head0 + a->H <= a->out_heads),
               "peer output needs int8 output, scale_peers, peer_rows % 128 == 0 and head0 + H <= out_heads");
    TB_REQUIRE(a->v_fp8 == nullptr || (a->v_scales != nullptr && a->dtype == TB_BF16 && sla_tc_supported(a)),
               "FP8 P/V needs bf16 inputs, v_scales and the tensor-core envelope");
    if (sla_tc_supported(a)) return sla_tc(a, st);
    TB_REQUIRE(a->lin_kv == nullptr, "fused linear epilogue needs the tensor-core envelope");
    return sla_simt(a, st);
}

// Which kernel tb_sla_attention would run for these arguments: 1 = the
// tcgen05 kernel, 0 = the CUDA-core kernel (tests assert the default
// configurations land on the tensor cores).
extern "C" int tb_sla_path(const tb_sla_args *a) { return (a != nullptr && sla_tc_supported(a)) ? 1 : 0; }

#ifdef TB_SLA_TRACE
extern "C" int tb_sla_trace_read(unsigned long long *host) {
    return cudaMemcpyFromSymbol(host, tb_sla_trace, sizeof(tb_sla_trace)) == cudaSuccess ? 0 : -2;
}
// phase[4] then sm[160][4]; reset = 1 re-arms the accumulators
extern "C" int tb_sla_phase_read(unsigned long long *host, int reset) {
    if (cudaMemcpyFromSymbol(host, tb_sla_phase, sizeof(tb_sla_phase)) != cudaSuccess) return -2;
    if (cudaMemcpyFromSymbol(host + 4, tb_sla_sm, sizeof(tb_sla_sm)) != cudaSuccess) return -2;
    if (reset) {
        static unsigned long long init[160][4];
        for (int i = 0; i < 160; i++) { init[i][0] = ~0ull; init[i][1] = 0; init[i][2] = ~0ull; init[i][3] = 0; }
        unsigned long long z[4] = {0, 0, 0, 0};
        if (cudaMemcpyToSymbol(tb_sla_phase, z, sizeof(z)) != cudaSuccess) return -2;
        if (cudaMemcpyToSymbol(tb_sla_sm, init, sizeof(init)) != cudaSuccess) return -2;
    }
    return 0;
}
#endif

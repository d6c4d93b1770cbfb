// sla_pipeline.cu -- the whole sla_attention (attention.py:392-421) behind one
// C-ABI call, for hosts that bind the library directly (SURVEY.md §8 b4
// `tb_sla_sage_fwd` / `tb_workspace_bytes`).  It issues exactly the sequence
// ops.sla_attention runs from Python on the tensor-core path:
//
//   side stream    k_mean (sequential chain) -> K codes (smoothed K; f32
//                  inputs: with the K pool, which top-k then waits for)
//   third stream   kv_part (per-block phi(K_b)^T [V_b | 1], linear branch;
//                  bf16 inputs: with the raw K pool + transposed copy)
//   caller stream  Q pool + codes -> [K pool (+ transposed copy)] -> top-k and
//                  the coverage matrix -> coverage GEMM (KV_sel) -> [q_block
//                  64: pair unions] -> fused tcgen05 attention
//
// The helper streams fork from and join back into the caller's stream with
// events, so the call is stream-ordered and CUDA-graph capturable.  Every
// intermediate lives in the caller's workspace (tb_sla_workspace_bytes); the
// library allocates nothing.
#include <cmath>
#include <mutex>

#include "common.cuh"

namespace tb {
namespace {

struct Layout {
    int64_t nq, nkv, count, ldt, ldc, dx, nt;
    bool f32, lin, q2;
    // byte offsets into the workspace
    int64_t kb, vb, km, qc, qs, qp, kc, ks, kp, kpt, idx, cov, kvp, kvsel, pidx, pcnt, total;
};

constexpr int64_t ALIGN = 256;
int64_t up(int64_t x) { return (x + ALIGN - 1) / ALIGN * ALIGN; }

bool make_layout(int64_t H, int64_t L, int64_t d, int64_t q_block, int64_t kv_block, double ratio, int dtype,
                 float linear_mix, Layout &o) {
    o.nq = cdiv(L, q_block);
    o.nkv = cdiv(L, kv_block);
    // attention.py:279 -- math.ceil(cfg.topk_ratio * num_kv) in IEEE double, as Python evaluates it
    o.count = (int64_t)std::ceil(ratio * (double)o.nkv);
    if (o.count < 1 || o.count > o.nkv) return false;
    o.ldt = cdiv(o.nkv, 4) * 4;
    o.ldc = cdiv(o.nkv, 8) * 8;
    o.dx = d + 1;
    while ((o.dx * d) % 256) o.dx++;
    o.nt = cdiv(o.nq, 2);
    o.f32 = dtype == TB_F32;
    o.lin = o.count < o.nkv && linear_mix != 0.0f;
    o.q2 = q_block == 64;
    int64_t off = 0;
    auto take = [&](int64_t bytes) { const int64_t at = off; off += up(bytes); return at; };
    const int64_t hld = H * L * d;
    o.kb = o.f32 ? take(hld * 2) : -1;                  // bf16 copies of f32 k, v (kv_part operands, V for PV)
    o.vb = o.f32 ? take(hld * 2) : -1;
    o.km = take(H * d * 4);
    o.qc = take(hld);
    o.qs = take(H * o.nq * 4);
    o.qp = take(H * o.nq * d * 4);
    o.kc = take(hld);
    o.ks = take(H * o.nkv * 4);
    o.kp = take(H * o.nkv * d * 4);
    o.kpt = take(H * d * o.ldt * 4);
    o.idx = take(H * o.nq * o.count * 4);
    o.cov = take(H * o.nq * o.ldc * 2);
    o.kvp = o.lin ? take(H * o.nkv * o.dx * d * 2) : -1;
    o.kvsel = o.lin ? take(H * o.nq * o.dx * d * 2) : -1;
    o.pidx = o.q2 ? take(H * o.nt * 2 * o.count * 4) : -1;
    o.pcnt = o.q2 ? take(H * o.nt * 4) : -1;
    o.total = off;
    return true;
}

bool envelope(int64_t L, int64_t d, int64_t q_block, int64_t kv_block, const Layout &o) {
    return d == 128 && kv_block == 64 && L >= 128 && o.count <= 2048 &&
           (q_block == 128 || (q_block == 64 && (2 * o.count < o.nkv ? 2 * o.count : o.nkv) <= 2048));
}

// per-device helper streams (created once, non-blocking)
cudaStream_t helper(int which) {
    static std::mutex m;
    static cudaStream_t s[64][2] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(m);
    if (dev < 0 || dev >= 64) return nullptr;
    if (!s[dev][which]) cudaStreamCreateWithFlags(&s[dev][which], cudaStreamNonBlocking);
    return s[dev][which];
}

}  // namespace
}  // namespace tb

using namespace tb;

extern "C" int64_t tb_sla_workspace_bytes(int64_t H, int64_t L, int64_t d, int64_t q_block, int64_t kv_block,
                                          double topk_ratio, float linear_mix, int dtype) {
    if (H < 0 || L < 1 || d < 1 || q_block < 1 || kv_block < 1 || !(topk_ratio > 0.0 && topk_ratio <= 1.0))
        return fail(TB_EINVAL, "bad shape or topk_ratio");
    Layout o;
    if (!make_layout(H, L, d, q_block, kv_block, topk_ratio, dtype, linear_mix, o)) return fail(TB_EINVAL, "bad count");
    return o.total;
}

extern "C" int tb_sla_forward(const void *q, const void *k, const void *v, int dtype, int64_t H, int64_t L, int64_t d,
                              int64_t q_block, int64_t kv_block, double topk_ratio, float linear_mix, float scale,
                              void *workspace, int64_t workspace_bytes, void *out, int out_dtype, void *stream) {
    TB_REQUIRE(dtype == TB_F32 || dtype == TB_BF16, "dtype must be f32 or bf16");
    TB_REQUIRE(out_dtype == TB_F32 || out_dtype == TB_BF16, "out dtype must be f32 or bf16");
    TB_REQUIRE(H >= 0 && L >= 1 && d >= 1, "bad shape");
    TB_REQUIRE(q_block >= 1 && kv_block >= 1 && q_block <= L && kv_block <= L, "block sizes exceed seq");
    TB_REQUIRE(topk_ratio > 0.0 && topk_ratio <= 1.0, "topk_ratio must be in (0, 1]");
    TB_REQUIRE(linear_mix >= 0.0f, "linear_mix must be >= 0");
    Layout o;
    TB_REQUIRE(make_layout(H, L, d, q_block, kv_block, topk_ratio, dtype, linear_mix, o), "bad count");
    if (!envelope(L, d, q_block, kv_block, o))
        return fail(TB_EUNSUPPORTED, "tb_sla_forward serves the tensor-core envelope (d 128, kv_block 64, q_block 128 or 64)");
    TB_REQUIRE(workspace != nullptr && workspace_bytes >= o.total, "workspace smaller than tb_sla_workspace_bytes");
    TB_REQUIRE(((uintptr_t)workspace % ALIGN) == 0, "workspace must be 256-byte aligned");
    if (H == 0) return TB_OK;
    uint8_t *w = reinterpret_cast<uint8_t *>(workspace);
    auto at = [&](int64_t off) -> void * { return off < 0 ? nullptr : w + off; };
    cudaStream_t main = as_stream(stream), side = helper(0), third = helper(1);
    TB_REQUIRE(side != nullptr && third != nullptr, "helper streams unavailable");
    int rc;
#define TB_CALL(expr)                                                                                       \
    do {                                                                                                    \
        if ((rc = (expr)) != TB_OK) return rc;                                                              \
    } while (0)
    // bf16 operands for f32 inputs (the kernels read V, and kv_part reads K and V, as bf16)
    const void *kb = k, *vb = v;
    if (o.f32) {
        TB_CALL(tb_cast_bf16((const float *)k, H * L * d, at(o.kb), stream));
        TB_CALL(tb_cast_bf16((const float *)v, H * L * d, at(o.vb), stream));
        kb = at(o.kb);
        vb = at(o.vb);
    }
    struct Events {                            // destroyed on every exit path
        cudaEvent_t e[3];
        Events() { for (auto &x : e) cudaEventCreateWithFlags(&x, cudaEventDisableTiming); }
        ~Events() { for (auto &x : e) cudaEventDestroy(x); }
    } ev;
    cudaEvent_t e0 = ev.e[0], e_side = ev.e[1], e_third = ev.e[2];
    cudaEventRecord(e0, main);
    cudaStreamWaitEvent(side, e0, 0);
    cudaStreamWaitEvent(third, e0, 0);
    float *km = (float *)at(o.km);
    // side: k_mean -> smoothed K codes (f32 inputs: the raw K pool in the same pass)
    TB_CALL(tb_kmean(k, dtype, H, L, d, km, side));
    TB_CALL(tb_pool_quant_tokens(k, dtype, km, H, L, d, kv_block, (int8_t *)at(o.kc), (float *)at(o.ks),
                                 o.f32 ? (float *)at(o.kp) : nullptr, side));
    cudaEventRecord(e_side, side);
    // third: the linear branch's per-block operand; bf16 inputs: with the raw K pool
    // and its transposed copy (the top-k operands) from the same tiles
    const bool kv_pool = o.lin && !o.f32;
    if (kv_pool)
        TB_CALL(tb_linear_kv_part_pool(kb, vb, H, L, d, kv_block, o.dx, at(o.kvp), (float *)at(o.kp),
                                       (float *)at(o.kpt), o.ldt, third));
    else if (o.lin)
        TB_CALL(tb_linear_kv_part(kb, vb, H, L, d, kv_block, o.dx, at(o.kvp), third));
    cudaEventRecord(e_third, third);
    // caller stream: pools, Q codes, top-k + coverage, coverage GEMM, fused kernel
    TB_CALL(tb_pool_quant_tokens(q, dtype, nullptr, H, L, d, q_block, (int8_t *)at(o.qc), (float *)at(o.qs),
                                 (float *)at(o.qp), stream));
    if (kv_pool) {
        cudaStreamWaitEvent(main, e_third, 0);   // the K pool came with kv_part
    } else if (!o.f32) {
        // bf16 without the linear branch: the raw K pool with its transposed copy, no k_mean wait
        TB_CALL(tb_pool_quant_tokens_t(k, dtype, nullptr, H, L, d, kv_block, nullptr, nullptr, (float *)at(o.kp),
                                       (float *)at(o.kpt), o.ldt, stream));
    } else {
        cudaStreamWaitEvent(main, e_side, 0);   // the K pool came with the K codes
    }
    TB_CALL(tb_topk_blocks_cov((const float *)at(o.qp), (const float *)at(o.kp),
                               o.f32 ? nullptr : (const float *)at(o.kpt), o.f32 ? 0 : o.ldt, H, o.nq, o.nkv, d,
                               o.count, (int32_t *)at(o.idx), nullptr, at(o.cov), o.ldc, stream));
    cudaStreamWaitEvent(main, e_third, 0);
    if (o.lin)
        TB_CALL(tb_gemm_bf16_batched(at(o.cov), at(o.kvp), at(o.kvsel), H, o.nq, o.dx * d, o.nkv, o.ldc, o.dx * d,
                                     o.dx * d, TB_BF16, stream));
    if (o.q2)
        TB_CALL(tb_pair_union((const int32_t *)at(o.idx), H, o.nq, o.count, (int32_t *)at(o.pidx),
                              (int32_t *)at(o.pcnt), 2 * o.count, stream));
    cudaStreamWaitEvent(main, e_side, 0);
    tb_sla_args a{};
    a.q = q; a.k = k; a.v = v; a.dtype = dtype;
    a.H = H; a.L = L; a.d = d; a.q_block = q_block; a.kv_block = kv_block; a.count = o.count;
    a.scale = scale; a.linear_mix = linear_mix; a.quantized = 1;
    a.q_codes = (const int8_t *)at(o.qc); a.k_codes = (const int8_t *)at(o.kc);
    a.q_scales = (const float *)at(o.qs); a.k_scales = (const float *)at(o.ks);
    a.k_mean = km; a.idx = (const int32_t *)at(o.idx);
    a.vt = o.f32 ? vb : nullptr; a.l_pad = o.nkv * 64;
    a.lin_kv = o.lin ? at(o.kvsel) : nullptr; a.lin_dx = o.dx;
    a.out = (float *)out; a.out_dtype = out_dtype;
    a.pair_idx = o.q2 ? (const int32_t *)at(o.pidx) : nullptr;
    a.pair_cnt = o.q2 ? (const int32_t *)at(o.pcnt) : nullptr;
    a.pair_ld = o.q2 ? 2 * o.count : 0;
    return tb_sla_attention(&a, stream);
#undef TB_CALL
}

// sla_simt.cu -- CUDA-core SLA sparse branch + combine for shapes outside
// the tensor-core kernel's envelope (any head_dim / block sizes; also the
// unquantized f32 branch).  Same semantics as the tcgen05 kernel:
//   _sparse_branch (attention.py:347-389): over the selected kv positions,
//     logits = scale*((prod*sq)*sk + q.k_mean) (quantized) or scale*(q.k),
//     online max/exp/sum with PV in f32;
//   combine (attention.py:410-421) with the linear branch num_l/den_l.
#include "common.cuh"

namespace tb {

template <typename T>
__global__ void __launch_bounds__(128) sla_simt_kernel(tb_sla_args a, int64_t nq, int64_t nkv) {
    extern __shared__ __align__(16) float sm[];
    const int64_t h = blockIdx.y, n = blockIdx.x;
    const int64_t d = a.d, L = a.L;
    const int64_t lo = n * a.q_block, hi = min(lo + a.q_block, L);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nwarps = blockDim.x >> 5;
    float *qrow = sm + warp * d;                 // per-warp query row (f32)
    const T *q = (const T *)a.q, *k = (const T *)a.k, *v = (const T *)a.v;
    const int32_t *sel = a.idx + (h * nq + n) * a.count;
    const float sq = a.quantized ? a.q_scales[h * nq + n] : 0.0f;
    constexpr int MAXC = 8;                       // d <= 256
    for (int64_t row = lo + warp; row < hi; row += nwarps) {
        const int64_t qoff = (h * L + row) * d;
        for (int64_t c = lane; c < d; c += 32) qrow[c] = to_f32(q[qoff + c]);
        __syncwarp();
        float corr = 0.0f;
        if (a.quantized) {
            // q_row . k_mean in f32 (a numpy matvec; tolerance-level term)
            float part = 0.0f;
            for (int64_t c = lane; c < d; c += 32) part = fmaf(qrow[c], a.k_mean[h * d + c], part);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
            corr = part;
        }
        float m = -INFINITY, l = 0.0f, acc[MAXC];
#pragma unroll
        for (int i = 0; i < MAXC; i++) acc[i] = 0.0f;
        for (int64_t s = 0; s < a.count; s++) {
            const int64_t b = sel[s];
            const int64_t k0 = b * a.kv_block, k1 = min(k0 + a.kv_block, L);
            const float sk = a.quantized ? a.k_scales[h * nkv + b] : 0.0f;
            for (int64_t base = k0; base < k1; base += 32) {
                const int64_t key = base + lane;
                float lg = -INFINITY;
                if (key < k1) {
                    if (a.quantized) {
                        const int8_t *qc = a.q_codes + (h * L + row) * d;
                        const int8_t *kc = a.k_codes + (h * L + key) * d;
                        int prod = 0;
                        for (int64_t c = 0; c < d; c++) prod += (int)qc[c] * (int)kc[c];
                        float approx = __fmul_rn(__fmul_rn((float)prod, sq), sk);
                        lg = __fmul_rn(a.scale, __fadd_rn(approx, corr));
                    } else {
                        float dot = 0.0f;
                        for (int64_t c = 0; c < d; c++) dot = fmaf(qrow[c], to_f32(k[(h * L + key) * d + c]), dot);
                        lg = __fmul_rn(a.scale, dot);
                    }
                }
                float cm = lg;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, o));
                const float mn = fmaxf(m, cm);
                const float alpha = (m == -INFINITY) ? 0.0f : __expf(m - mn);
                const float p = (key < k1) ? __expf(lg - mn) : 0.0f;
                float ps = p;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
                l = l * alpha + ps;
#pragma unroll
                for (int i = 0; i < MAXC; i++) acc[i] *= alpha;
                const int nk = (int)imin64(32, k1 - base);
                for (int j = 0; j < nk; j++) {
                    const float pj = __shfl_sync(0xffffffffu, p, j);
                    const T *vr = v + (h * L + base + j) * d;
#pragma unroll
                    for (int i = 0; i < MAXC; i++) {
                        const int64_t c = lane + 32 * i;
                        if (c < d) acc[i] = fmaf(pj, to_f32(vr[c]), acc[i]);
                    }
                }
                m = mn;
            }
        }
        // combine with the linear branch (attention.py:410-421)
        const bool lin = a.num_l != nullptr && a.linear_mix != 0.0f;
        const float *nl_row = nullptr;
        float ss = 1.0f, shrink = 0.0f, dl = 0.0f;
        if (lin) {
            const float ref = fmaxf(m, 0.0f);
            ss = expf(m - ref);
            shrink = expf(-ref) * a.linear_mix;
            if (a.lin_ld) {
                nl_row = a.num_l + h * a.lin_hs + row * a.lin_ld;
                dl = nl_row[d];
            } else {
                nl_row = a.num_l + (h * L + row) * d;
                dl = a.den_l[h * L + row];
            }
        }
        const float den = lin ? (l * ss + shrink * dl) : l;
#pragma unroll
        for (int i = 0; i < MAXC; i++) {
            const int64_t c = lane + 32 * i;
            if (c < d) {
                float num = lin ? (acc[i] * ss + shrink * nl_row[c]) : acc[i];
                float o = num / den;
                if (a.out_dtype == TB_BF16)
                    reinterpret_cast<__nv_bfloat16 *>(a.out)[(h * L + row) * d + c] = __float2bfloat16_rn(o);
                else
                    a.out[(h * L + row) * d + c] = o;
            }
        }
        if (lane == 0) {
            if (a.row_max) a.row_max[h * L + row] = m;
            if (a.den) a.den[h * L + row] = l;
        }
        __syncwarp();
    }
}

int sla_simt(const tb_sla_args *a, cudaStream_t st) {
    TB_REQUIRE(a->d <= 256, "head_dim > 256 unsupported");
    const int64_t nq = cdiv(a->L, a->q_block), nkv = cdiv(a->L, a->kv_block);
    dim3 grid((unsigned)nq, (unsigned)a->H);
    size_t smem = 4 * a->d * sizeof(float);
    if (a->dtype == TB_F32) sla_simt_kernel<float><<<grid, 128, smem, st>>>(*a, nq, nkv);
    else sla_simt_kernel<__nv_bfloat16><<<grid, 128, smem, st>>>(*a, nq, nkv);
    return check_launch("sla_simt");
}

}  // namespace tb

// linear_simt.cu -- the linear-attention branch (attention.py:287-335) on CUDA
// cores for shapes outside the tcgen05 envelope (head_dim != 128, kv_block !=
// 64, unquantized branch, the unmasked linear_attention of one block of L
// tokens).  f32 throughout, three passes, caller-allocated workspaces:
//   kv_part[h,b] = phi(K_b)^T [V_b | 1]           [H, nkv, d, d+1]  (:320-325)
//   kv_sel[h,n]  = sum_{b in complement(n)} kv_part[h,b]   [H, nq, d, d+1]  (:326-328)
//   out[h,row]   = phi(q_row) . kv_sel[h, n(row)]  [H, nq*q_block, dx] (:329-334)
// out columns 0..d-1 are the numerator, column d the denominator.
#include "common.cuh"

namespace tb {
namespace {

__device__ __forceinline__ float phi(float x) { return x >= 0.0f ? x + 1.0f : expf(x); }

template <typename T>
__device__ __forceinline__ float ld(const T *p) { return to_f32(*p); }

constexpr int CH = 16;   // tokens per shared-memory chunk

template <typename T>
__global__ void __launch_bounds__(256) lin_kv_part_kernel(const T *__restrict__ k, const T *__restrict__ v, int64_t L,
                                                          int d, int kv_block, int nkv, float *__restrict__ part) {
    extern __shared__ float sm[];
    float *pk = sm;                      // [CH][d]
    float *vv = sm + CH * d;             // [CH][d + 1]
    const int b = blockIdx.x, h = blockIdx.y;
    const int dx = d + 1;
    const int64_t t0 = (int64_t)b * kv_block;
    const int64_t t1 = t0 + kv_block < L ? t0 + kv_block : L;
    const int nout = d * dx;
    float acc[8];
    const int per = (nout + blockDim.x - 1) / blockDim.x;          // outputs per thread (<= 8 for d <= 44 ... )
    for (int base = 0; base < per; base += 8) {
#pragma unroll
        for (int u = 0; u < 8; u++) acc[u] = 0.0f;
        for (int64_t tc = t0; tc < t1; tc += CH) {
            const int n = (int)((t1 - tc) < CH ? (t1 - tc) : CH);
            __syncthreads();
            for (int i = threadIdx.x; i < n * d; i += blockDim.x) {
                const int tt = i / d, c = i % d;
                const int64_t off = ((int64_t)h * L + tc + tt) * d + c;
                pk[tt * d + c] = phi(ld(k + off));
                vv[tt * dx + c] = ld(v + off);
            }
            for (int i = threadIdx.x; i < n; i += blockDim.x) vv[i * dx + d] = 1.0f;
            __syncthreads();
#pragma unroll
            for (int u = 0; u < 8; u++) {
                const int o = (base + u) * blockDim.x + threadIdx.x;
                if (base + u < per && o < nout) {
                    const int c = o / dx, j = o % dx;
                    float a = acc[u];
                    for (int tt = 0; tt < n; tt++) a = fmaf(pk[tt * d + c], vv[tt * dx + j], a);
                    acc[u] = a;
                }
            }
        }
#pragma unroll
        for (int u = 0; u < 8; u++) {
            const int o = (base + u) * blockDim.x + threadIdx.x;
            if (base + u < per && o < nout) part[(((int64_t)h * nkv + b) * nout) + o] = acc[u];
        }
    }
}

__global__ void __launch_bounds__(256) lin_kv_sel_kernel(const float *__restrict__ part, const uint8_t *__restrict__ comp,
                                                         int nq, int nkv, int nout, float *__restrict__ sel) {
    const int n = blockIdx.x, h = blockIdx.y;
    const uint8_t *cr = comp ? comp + ((int64_t)h * nq + n) * nkv : nullptr;
    for (int o = threadIdx.x + blockIdx.z * blockDim.x; o < nout; o += blockDim.x * gridDim.z) {
        float a = 0.0f;
        for (int b = 0; b < nkv; b++)
            if (!cr || cr[b]) a += part[((int64_t)h * nkv + b) * nout + o];
        sel[((int64_t)h * nq + n) * nout + o] = a;
    }
}

template <typename T>
__global__ void __launch_bounds__(256) lin_out_kernel(const T *__restrict__ q, const float *__restrict__ sel, int64_t L,
                                                      int d, int q_block, int nq, int64_t lq, int dx_out,
                                                      float *__restrict__ out) {
    extern __shared__ float pq[];        // [rows][d] phi(q) of this CTA's rows
    const int h = blockIdx.y;
    const int64_t r0 = (int64_t)blockIdx.x * 8;
    const int dx = d + 1;
    for (int i = threadIdx.x; i < 8 * d; i += blockDim.x) {
        const int64_t row = r0 + i / d;
        pq[i] = row < L ? phi(ld(q + ((int64_t)h * L + row) * d + i % d)) : 0.0f;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 8 * dx_out; i += blockDim.x) {
        const int rr = i / dx_out, j = i % dx_out;
        const int64_t row = r0 + rr;
        if (row >= lq) continue;
        float a = 0.0f;
        if (j < dx) {
            const float *s = sel + ((int64_t)h * nq + row / q_block) * (int64_t)d * dx + j;
            for (int c = 0; c < d; c++) a = fmaf(pq[rr * d + c], s[(int64_t)c * dx], a);
        }
        out[((int64_t)h * lq + row) * dx_out + j] = a;
    }
}

}  // namespace
}  // namespace tb

using namespace tb;

extern "C" int tb_linear_branch_simt(const void *q, const void *k, const void *v, int dtype, int64_t H, int64_t L,
                                     int64_t d, const uint8_t *comp, int64_t nq, int64_t nkv, int64_t q_block,
                                     int64_t kv_block, float *kv_part_ws, float *kv_sel_ws, float *out, int64_t dx_out,
                                     void *stream) {
    TB_REQUIRE(dtype == TB_F32 || dtype == TB_BF16, "dtype must be f32 or bf16");
    TB_REQUIRE(d >= 1 && d <= 256 && dx_out >= d + 1, "head_dim in [1, 256], dx_out >= d + 1");
    TB_REQUIRE(nkv == cdiv(L, kv_block) && nq * q_block >= L, "block counts do not cover the sequence");
    TB_REQUIRE(kv_part_ws && kv_sel_ws && out, "workspaces and output required");
    if (H == 0) return TB_OK;
    cudaStream_t st = as_stream(stream);
    const int nout = (int)(d * (d + 1));
    const size_t sm1 = (size_t)CH * (2 * d + 1) * 4;
    dim3 g1((unsigned)nkv, (unsigned)H);
    if (dtype == TB_F32) {
        smem_attr(lin_kv_part_kernel<float>, (int)sm1);
        lin_kv_part_kernel<float><<<g1, 256, sm1, st>>>((const float *)k, (const float *)v, L, (int)d, (int)kv_block,
                                                        (int)nkv, kv_part_ws);
    } else {
        smem_attr(lin_kv_part_kernel<__nv_bfloat16>, (int)sm1);
        lin_kv_part_kernel<__nv_bfloat16><<<g1, 256, sm1, st>>>((const __nv_bfloat16 *)k, (const __nv_bfloat16 *)v, L,
                                                                (int)d, (int)kv_block, (int)nkv, kv_part_ws);
    }
    dim3 g2((unsigned)nq, (unsigned)H, (unsigned)cdiv(nout, 256));
    lin_kv_sel_kernel<<<g2, 256, 0, st>>>(kv_part_ws, comp, (int)nq, (int)nkv, nout, kv_sel_ws);
    const int64_t lq = nq * q_block;
    dim3 g3((unsigned)cdiv(lq, 8), (unsigned)H);
    const size_t sm3 = (size_t)8 * d * 4;
    if (dtype == TB_F32)
        lin_out_kernel<float><<<g3, 256, sm3, st>>>((const float *)q, kv_sel_ws, L, (int)d, (int)q_block, (int)nq, lq,
                                                    (int)dx_out, out);
    else
        lin_out_kernel<__nv_bfloat16><<<g3, 256, sm3, st>>>((const __nv_bfloat16 *)q, kv_sel_ws, L, (int)d,
                                                            (int)q_block, (int)nq, lq, (int)dx_out, out);
    return check_launch("linear_branch_simt");
}

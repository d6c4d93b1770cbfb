/*
 * tb_capi.h -- C ABI of the B200 (sm_100a) TurboDiffusion hot path.
 *
 * Every entry point is extern "C", takes plain device pointers, int64 sizes
 * and a cudaStream_t passed as void*, is stream-ordered and asynchronous,
 * allocates nothing (callers own every output and workspace), and returns
 * 0 on success or a negative TB_E* code; tb_last_error() returns the
 * thread-local message of the last failure.
 *
 * Each function names the reference operator it replaces
 * (/root/reference/pkg/src/turbobench/<file>:<line>).  The Python drop-in
 * modules (paper_2512_16093_b200/{attention,blockquant,sampler}.py) are the
 * reference-facing binding; INTEGRATION.md shows the ctypes binding a
 * turbobench maintainer would add.
 */
#ifndef TB_CAPI_H
#define TB_CAPI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum tb_status {
    TB_OK = 0,
    TB_EINVAL = -1,      /* bad shape / argument (Python: ValueError) */
    TB_ECUDA = -2,       /* CUDA runtime / launch failure (RuntimeError) */
    TB_EUNSUPPORTED = -3 /* shape outside the kernel's envelope */
};

enum tb_dtype { TB_F32 = 0, TB_BF16 = 1, TB_I8 = 2 };

const char *tb_last_error(void);
/* 1 when the library was built for sm_100a and a capable device is visible. */
int tb_device_ok(void);
const char *tb_build_info(void);

/* ---------------------------------------------------------------- quant */

/* blockquant.quantize_blockwise (blockquant.py:91-110): symmetric absmax
 * INT8 codes per block x block tile, scale = absmax/127 (IEEE RN), code =
 * clip(rint(x/scale)) with zero tiles -> scale 0, codes 0.  x is [rows,cols]
 * row-major f32 or bf16; q int8 [rows,cols]; scales f32 [ceil(r/b),ceil(c/b)].
 * *nonfinite (device int, may be NULL) is set to 1 if any input is inf/nan
 * (the reference raises ValueError, blockquant.py:103-104). */
int tb_quantize_blockwise(const void *x, int dtype, int64_t rows, int64_t cols, int64_t block,
                          int8_t *q, float *scales, int32_t *nonfinite, void *stream);

/* blockquant.dequantize_blockwise (blockquant.py:113-116). */
int tb_dequantize_blockwise(const int8_t *q, const float *scales, int64_t rows, int64_t cols,
                            int64_t block, float *out, void *stream);

/* Transposes weight codes [K,N] -> [N,K] (the K-major B operand layout of
 * the tensor-core GEMM).  Done once per weight at load time. */
int tb_transpose_codes(const int8_t *src, int64_t rows, int64_t cols, int8_t *dst, void *stream);

/* blockquant.w8a8_matmul + quantized_linear_forward bias add
 * (blockquant.py:132-161, 164-182).  a: codes [M,K] + scales [ceil(M/b),ceil(K/b)];
 * b: TRANSPOSED weight codes bt [N,K] + scales [ceil(K/b),ceil(N/b)] (the
 * reference's [K,N] weight, transposed once).  out[M,N] (f32 or bf16) =
 * sum over k-blocks ascending of (exact_int_segment * sa) * sb, then + bias
 * (f32 [N], may be NULL).  block==128, K%128==0, N%16==0 runs on tcgen05
 * (kind::i8, s32 TMEM accumulators); other shapes on a CUDA-core kernel with
 * the identical arithmetic.  Any block with block * 127^2 < 2^31: segments
 * are exact int32 sums rounded to f32 once, which is what the reference's
 * int64 path does above block 1040 (blockquant.py:119-129). */
int tb_w8a8_gemm(const int8_t *a, const float *sa, const int8_t *bt, const float *sb,
                 const float *bias, int64_t M, int64_t N, int64_t K, int64_t block,
                 void *out, int out_dtype, void *stream);

/* Fused activation quantization + W8A8 GEMM (quantized_linear_forward,
 * blockquant.py:164-182): x [M,K] f32/bf16 is block-quantized into the
 * caller's workspace (xq [M,K] int8, xs scales) then multiplied. */
int tb_quantized_linear(const void *x, int x_dtype, const int8_t *bt, const float *sb,
                        const float *bias, int64_t M, int64_t N, int64_t K, int64_t block,
                        int8_t *xq_ws, float *xs_ws, void *out, int out_dtype, void *stream);

/* ------------------------------------------------------- SLA importance */

/* attention.pool_block_means (attention.py:256-266), numpy pairwise order:
 * out[h,b,c] = (x[lo] + pairwise(x[lo+1:lo+e])) / f32(e).  x [H,L,d]. */
int tb_pool_block_means(const void *x, int dtype, int64_t H, int64_t L, int64_t d, int64_t block,
                        float *out, void *stream);

/* smooth_keys k_mean (attention.py:179-188): sequential f32 chain over
 * tokens per (h, channel), / f32(L).  k [H,L,d] -> kmean [H,d]. */
int tb_kmean(const void *k, int dtype, int64_t H, int64_t L, int64_t d, float *kmean, void *stream);

/* _quantize_token_blocks (attention.py:201-220) of x - center (center
 * [H,d] may be NULL: Q path; k_mean: K path), optionally fused with the
 * block pooling of the RAW x (pooled may be NULL).  codes int8 [H,L,d],
 * scales f32 [H,ceil(L/block)]. */
int tb_pool_quant_tokens(const void *x, int dtype, const float *center, int64_t H, int64_t L,
                         int64_t d, int64_t block, int8_t *codes, float *scales, float *pooled,
                         void *stream);

/* select_topk_blocks + BlockMask.complement (attention.py:269-284,
 * 122-132): scores = qp.kp^T in the reference's OpenBLAS order, top-count
 * per row with ties to the lower index, ascending.  idx int32
 * [H,nq,count]; comp (may be NULL) uint8 [H,nq,nkv] = 1 for blocks NOT
 * selected; scores_out (may be NULL) f32 [H,nq,nkv]. */
int tb_topk_blocks(const float *qp, const float *kp, int64_t H, int64_t nq, int64_t nkv,
                   int64_t d, int64_t count, int32_t *idx, uint8_t *comp, float *scores_out,
                   void *stream);

/* tb_pool_quant_tokens plus a transposed copy of the pooled means,
 * pooled_t [H, d, ldt] (ldt >= blocks): the coalesced kp operand of
 * tb_topk_blocks_cov. */
int tb_pool_quant_tokens_t(const void *x, int dtype, const float *center, int64_t H, int64_t L, int64_t d,
                           int64_t block, int8_t *codes, float *scales, float *pooled, float *pooled_t,
                           int64_t ldt, void *stream);

/* tb_topk_blocks plus the complement written as the bf16 coverage matrix
 * cov [H, nq, cov_ld] (1.0 = kv block in the complement, padding columns
 * 0) -- the A operand of the linear branch's GEMM (attention.py:326-328).
 * kpt (optional, from tb_pool_quant_tokens_t, row pitch ldk) enables the
 * coalesced fast path.  comp may be NULL. */
int tb_topk_blocks_cov(const float *qp, const float *kp, const float *kpt, int64_t ldk, int64_t H, int64_t nq,
                       int64_t nkv, int64_t d, int64_t count, int32_t *idx, uint8_t *comp, void *cov,
                       int64_t cov_ld, void *stream);

/* ------------------------------------------------------- SLA attention */

typedef struct tb_sla_args {
    /* raw inputs [H,L,d] (dtype f32 or bf16) */
    const void *q, *k, *v;
    int dtype;
    int64_t H, L, d, q_block, kv_block, count;
    float scale;            /* logit scale (1/sqrt(d) default) */
    float linear_mix;       /* attention.py:416-421 */
    int quantized;          /* SLAConfig.quantized_sparse_branch */
    /* prepared operands (from the prep entry points above) */
    const int8_t *q_codes, *k_codes;   /* [H,L,d] */
    const float *q_scales, *k_scales;  /* [H,nq], [H,nkv] */
    const float *k_mean;               /* [H,d] */
    const int32_t *idx;                /* [H,nq,count] ascending */
    const void *vt;                    /* bf16 copy of V [H,L,d] for the tensor-core path when
                                          dtype is f32 (ignored for bf16 inputs: v is read directly) */
    int64_t l_pad;                     /* unused (kept for ABI stability) */
    /* linear branch over the complement (may be NULL -> no linear term) */
    const float *num_l, *den_l;        /* [H,L,d], [H,L] */
    /* packed linear branch: when lin_ld != 0, row r of head h is
     * num_l + h*lin_hs + r*lin_ld (d numerators followed by the
     * denominator at column d; den_l is ignored) */
    int64_t lin_ld, lin_hs;
    /* fused linear branch (tensor-core path): when lin_kv != NULL, the
     * kernel computes num_l = phi(Q) . KV_sel^T itself as one more tcgen05
     * MMA in its epilogue.  lin_kv is bf16 [H, nq, lin_dx, d]: rows 0..d-1 of
     * q-block n hold KV_sel[n]^T (= sum over complement blocks of
     * V_b^T phi(K_b)), row d holds sum phi(K_b) (the denominator vector). */
    const void *lin_kv;
    int64_t lin_dx;
    /* outputs */
    float *out;                        /* [H,L,d] f32 (or bf16 when out_dtype) */
    int out_dtype;
    float *row_max, *den;              /* optional [H,L] sparse-branch stats */
    /* out_dtype == TB_I8 (tensor-core path, no row_max / den): out holds the
     * block-quantized bf16-rounded output as the out-projection's A operand --
     * int8 codes [L, H*d] row-major (token, head*d + channel) -- and
     * out_scales [ceil(L/128), H] its 128 x 128 block scales (one per
     * (q-block, head) tile; quantize_blockwise_planar semantics) */
    float *out_scales;
    /* FP8 P/V (opt-in; tensor-core path, bf16 inputs): when
     * v_fp8 != NULL the PV product runs as kind::f8f6f4 on e4m3 P and the e4m3
     * V codes [H,L,d] from tb_quant_v_fp8 with their per-head scales v_scales
     * [H]; NULL keeps BF16 P/V (the default: FP8 misses rel-L1 <= 1e-2 on
     * sparse-dominated rows). */
    const uint8_t *v_fp8;
    const float *v_scales;
    /* Fused Ulysses return path (out_dtype TB_I8 only):
     * when out_peers != NULL the epilogue stores each 128-token tile's int8
     * codes and block scale straight into the buffers of the rank that owns
     * those tokens (NVLink peer memory from tb_peer_alloc / tb_peer_import), instead
     * of a local buffer followed by an all-to-all.  out_peers / scale_peers
     * are DEVICE arrays of P pointers; owner = row / peer_rows (peer_rows %
     * 128 == 0); codes land at out_peers[owner] + (row - owner*peer_rows) *
     * out_heads*d + (head0 + h)*d and the scale at scale_peers[owner]
     * [((row - owner*peer_rows)/128) * out_heads + head0 + h].  out and
     * out_scales are ignored. */
    void *const *out_peers;
    float *const *scale_peers;
    int64_t peer_rows, head0, out_heads;
    /* q_block 64 (the reference default, SLAConfig / QuantAttnConfig) on the
     * tensor-core kernel: 128-row tiles of two q-blocks walk the union of
     * their top-k lists, from tb_pair_union (pair_idx [H, ceil(nq/2),
     * pair_ld], pair_cnt [H, ceil(nq/2)]).  NULL keeps q_block 64 on the
     * CUDA-core kernel. */
    const int32_t *pair_idx, *pair_cnt;
    int64_t pair_ld;
} tb_sla_args;

/* _sparse_branch + combine (attention.py:347-389, 392-421).  d==128,
 * q_block 128 (or 64 with pair_idx), kv_block==64, quantized -> tcgen05 kernel (INT8 QK^T with
 * s32 TMEM accumulators, BF16 PV with f32 TMEM accumulators, TMA/bulk
 * staged tiles, warp-specialised online softmax); other shapes -> CUDA-core
 * kernel with the same semantics. */
int tb_sla_attention(const tb_sla_args *a, void *stream);

/* Union of the top-k lists of q-block pairs (2t, 2t+1) for the q_block 64
 * tensor-core attention (tb_sla_args.pair_idx): idx [H, nq, count]
 * ascending (select_topk_blocks, attention.py:269-284) -> per tile t the
 * ascending distinct kv blocks of both lists, entry = block | (mask << 28)
 * with mask bit 0 = selected by q-block 2t, bit 1 = by 2t+1; pair_cnt = the
 * entries per tile (count <= pair_cnt <= 2*count).  pair_ld >= 2*count. */
/* linear_attention (attention.py:287-335) on CUDA cores, f32, for shapes
 * outside the tensor-core envelope: kv_part_ws [H, nkv, d, d+1] = per kv
 * block phi(K_b)^T [V_b | 1]; kv_sel_ws [H, nq, d, d+1] = its sum over the
 * complement blocks of each q-block (comp uint8 [H, nq, nkv], 1 = block in
 * the complement; NULL = every block, the unmasked form with nq = nkv = 1,
 * q_block = kv_block = L); out [H, nq*q_block, dx_out] f32 = phi(q_row) .
 * kv_sel (columns 0..d-1 numerator, column d denominator, the rest 0). */
int tb_linear_branch_simt(const void *q, const void *k, const void *v, int dtype, int64_t H, int64_t L,
                          int64_t d, const uint8_t *comp, int64_t nq, int64_t nkv, int64_t q_block,
                          int64_t kv_block, float *kv_part_ws, float *kv_sel_ws, float *out, int64_t dx_out,
                          void *stream);

/* ---------------------------------------------- Ulysses exchange (NCCL)
 * (no reference function -- the reference is
 * single-process).  Token shard x [L_p, H, d] (rank r owns
 * tokens [r*per, min((r+1)*per, L)), per = tb_ulysses_shard(L, P, align))
 * -> head shard out [H/P, L, d] (heads [r*H/P, (r+1)*H/P)), and back.
 * Elements are esize bytes (bf16 2, int8 1, f32 4; d*esize % 16 == 0).
 * send_ws / recv_ws: caller-allocated, tb_ulysses_workspace_bytes each,
 * layout [P, per, H/P, d].  comm: the caller's ncclComm_t (one grouped
 * ncclSend/ncclRecv per peer; NULL allowed when P == 1).  stages: TB_UL_PACK
 * | TB_UL_EXCHANGE | TB_UL_UNPACK (TB_UL_ALL for the whole op; the pieces let a
 * host run the exchange itself).  Stream-ordered. */
#define TB_UL_PACK 1
#define TB_UL_EXCHANGE 2
#define TB_UL_UNPACK 4
#define TB_UL_ALL 7
int64_t tb_ulysses_shard(int64_t L, int64_t P, int64_t align);
int64_t tb_ulysses_workspace_bytes(int64_t L, int64_t H, int64_t d, int64_t esize, int64_t P, int64_t align);
int tb_ulysses_seq_to_heads(const void *x, int64_t L, int64_t H, int64_t d, int64_t esize, int64_t P,
                            int64_t rank, int64_t align, void *send_ws, void *recv_ws, void *out,
                            void *comm, int stages, void *stream);
int tb_ulysses_heads_to_seq(const void *o, int64_t L, int64_t H, int64_t d, int64_t esize, int64_t P,
                            int64_t rank, int64_t align, void *send_ws, void *recv_ws, void *out,
                            void *comm, int stages, void *stream);
/* NCCL communicator helpers for C-ABI hosts (libnccl.so.2 resolved at run
 * time): a 128-byte ncclUniqueId made on one rank and shared by the host's
 * own means, then one communicator per rank. */
int tb_nccl_unique_id(void *id128);
int tb_nccl_comm_init(void **comm, const void *id128, int64_t nranks, int64_t rank);
int tb_nccl_comm_destroy(void *comm);

/* The whole sla_attention (attention.py:392-421) in one stream-ordered call
 * (SURVEY.md §8 b4 tb_sla_sage_fwd): k_mean and the smoothed K codes, the Q
 * pool + codes, the K pool, the top-k selection and coverage matrix, the
 * linear branch's kv_part and coverage GEMM, the q_block-64 pair unions, and
 * the fused tcgen05 kernel -- the sequence ops.sla_attention issues, with two
 * internal helper streams forked from and joined back into `stream` by events
 * (graph-capturable).  count = ceil(topk_ratio * num_kv) in double precision
 * (attention.py:279).  Every intermediate lives in `workspace` (256-byte
 * aligned, at least tb_sla_workspace_bytes(...) bytes, SURVEY b4
 * tb_workspace_bytes); nothing is allocated.  Tensor-core envelope only (d 128,
 * kv_block 64, q_block 128 or 64, quantized branch): TB_EUNSUPPORTED otherwise.
 * q, k, v [H, L, d] f32 or bf16; out [H, L, d] f32 or bf16. */
int64_t tb_sla_workspace_bytes(int64_t H, int64_t L, int64_t d, int64_t q_block, int64_t kv_block, double topk_ratio,
                               float linear_mix, int dtype);
int tb_sla_forward(const void *q, const void *k, const void *v, int dtype, int64_t H, int64_t L, int64_t d,
                   int64_t q_block, int64_t kv_block, double topk_ratio, float linear_mix, float scale,
                   void *workspace, int64_t workspace_bytes, void *out, int out_dtype, void *stream);

/* 1 when tb_sla_attention would run these arguments on the tcgen05 kernel,
 * 0 for the CUDA-core kernel. */
int tb_sla_path(const tb_sla_args *a);

/* f32 -> bf16 (round to nearest even) copy of n elements: the bf16 V operand
 * (tb_sla_args.vt) when the attention inputs are f32. */
int tb_cast_bf16(const float *x, int64_t n, void *y, void *stream);

/* HOST staging for host-array callers (replaces the implicit numpy -> f32
 * conversion of AttnInputs, attention.py:38-60, on the upload side): copies n
 * elements of src into dst (normally page-locked), src_dtype -> dst_dtype in
 * {F32->F32, BF16->BF16, I8->I8, F32->BF16 (round to nearest even)}, on a
 * persistent pool of nthreads host threads (<= 0: TB_HOST_THREADS or every
 * hardware thread; fixed at the first call) with non-temporal stores.
 * Synchronous; no device work. */
int tb_host_stage(void *dst, const void *src, int64_t n, int src_dtype, int dst_dtype, int64_t nthreads);
int64_t tb_host_threads(void);

/* Lossless narrow upload encoding for the same staging step: when every one of
 * the n f32 values in src is exactly representable in bf16 (low 16 bits zero --
 * activations of a bf16 model handed over as f32 arrays), writes their bf16
 * bit patterns to dst and returns 1; otherwise returns 0 and dst is
 * unspecified (the caller stages f32).  The device widens bf16 -> f32
 * exactly, so the kernels see the caller's f32 values either way. */
int tb_host_stage_bf16_exact(void *dst, const float *src, int64_t n, int64_t nthreads);

/* Instrumentation: writes the device %globaltimer (ns) to *dst when the
 * one-thread kernel runs on `stream` (graph-capturable stream timeline). */
int tb_timestamp(unsigned long long *dst, void *stream);

int tb_pair_union(const int32_t *idx, int64_t H, int64_t nq, int64_t count, int32_t *pair_idx,
                  int32_t *pair_cnt, int64_t pair_ld, void *stream);

/* ---------------------------------------------- NVLink peer memory
 * (new, multi-GPU: the fused Ulysses exchanges store into peers' buffers).
 * tb_peer_alloc: a dedicated cudaMalloc (zeroed) that CUDA IPC can export;
 * tb_peer_export writes its 64-byte cudaIpcMemHandle_t, tb_peer_import maps
 * a peer's handle into this process (cudaIpcMemLazyEnablePeerAccess).
 * tb_peer_barrier: stream-ordered device barrier of a group of P ranks over
 * per-rank flag blocks (P uint32 each, in peer memory; flags = DEVICE array
 * of the P block pointers): barrier number `epoch` (monotonic, starting at
 * 1) makes every peer's stores issued before its barrier visible to the
 * work after this rank's. */
int tb_peer_alloc(int64_t bytes, void **ptr);
int tb_peer_free(void *ptr);
int tb_peer_export(void *ptr, void *handle);
int tb_peer_import(const void *handle, void **ptr);
int tb_peer_close(void *ptr);
int tb_peer_barrier(uint32_t *const *flags, int64_t P, int64_t rank, uint32_t epoch, void *stream);

/* FP8 V for the opt-in FP8 P/V path (no reference function; SURVEY.md §8
 * a17).  Per head h: scale[h] = f32(absmax(v[h])) / 448 (RN), codes =
 * e4m3 round-to-nearest-even, satfinite, of v / safe (IEEE divide; safe = 1
 * when the head is all zero).  am_ws: H uint32 of workspace.  Restated in
 * oracle/oracle.py quantize_v_fp8. */
int tb_quant_v_fp8(const void *v, int dtype, int64_t H, int64_t L, int64_t d, uint8_t *codes, float *scales,
                   unsigned *am_ws, void *stream);

/* V [H,L,d] -> bf16 V^T [H,d,l_pad] (zero padded), the K-major B operand
 * of the PV MMA. */
int tb_transpose_v(const void *v, int dtype, int64_t H, int64_t L, int64_t d, int64_t l_pad,
                   void *vt, void *stream);

/* Feature map phi (attention.py:287-290) of x [H,L,d] into a padded GEMM
 * operand out [H,l_pad,d] (f32 or bf16); rows t >= L are ZERO (not phi(0)),
 * so padded kv blocks contribute nothing to phi(K)^T V (attention.py:320-325). */
int tb_feature_map(const void *x, int dtype, int64_t H, int64_t L, int64_t d, int64_t l_pad,
                   void *out, int out_dtype, void *stream);

/* Linear-branch and PV operands in one pass over q, k, v
 * (attention.py:306-325): phiq [H,lq,d] = phi(q), phik [H,lk,d] = phi(k)
 * (rows >= L zero), vext [H,lk,dx] = [v | 1 | 0..] so that phi(K_b)^T vext
 * carries both phi(K_b)^T V_b and sum phi(K_b) (column d), and the bf16
 * V^T [H,d,lvt] B operand of the PV MMA.  Any of phiq / phik(+vext) / vt may
 * be NULL.  out_dtype bf16 or f32; d % 8 == 0, dx % 8 == 0, dx > d. */
int tb_linear_operands(const void *q, const void *k, const void *v, int dtype, int64_t H, int64_t L,
                       int64_t d, int64_t lq, int64_t lk, int64_t dx, void *phiq, void *phik,
                       void *vext, int out_dtype, void *vt, int64_t lvt, void *stream);

/* Batched bf16 GEMM on tcgen05 (f32 accumulate): for each h < H,
 * C[h] (MxN) = A[h] (MxK, row pitch lda, K contiguous) . B[h] (KxN, row
 * pitch ldb, N contiguous); C row pitch ldc, bf16 or f32.  N % 256 == 0.
 * Used for the linear branch's coverage GEMM kv_sel = cov . kv_part
 * (attention.py:326-328). */
int tb_gemm_bf16_batched(const void *A, const void *B, void *C, int64_t H, int64_t M, int64_t N,
                         int64_t K, int64_t lda, int64_t ldb, int64_t ldc, int out_dtype, void *stream);

/* Per-kv-block linear-branch operand (attention.py:320-325) straight from
 * bf16 k, v [H,L,d] on tcgen05: kv_part [H, nkv, dx, d] bf16 with rows
 * 0..d-1 = V_b^T phi(K_b), row d = sum_t phi(K_b), rows d+1.. zero (padded
 * tokens contribute nothing).  d == 128, kv_block == 64, dx*d % 256 == 0.
 * Replaces linear_attention's per-block einsums (attention.py:322-325). */
int tb_linear_kv_part(const void *k, const void *v, int64_t H, int64_t L, int64_t d, int64_t kv_block,
                      int64_t dx, void *kv_part, void *stream);

/* tb_linear_kv_part that also writes the raw K block means kp [H, nkv, d] f32
 * (pool_block_means of k, attention.py:256-266, numpy's reduceat order,
 * bit-exact) and, when kpt != NULL, their transposed copy kpt [H, d, ldt]
 * (ldt >= nkv) -- the operands of tb_topk_blocks_cov -- from the K tiles the
 * kernel already holds: no separate K pooling pass. */
int tb_linear_kv_part_pool(const void *k, const void *v, int64_t H, int64_t L, int64_t d, int64_t kv_block,
                           int64_t dx, void *kv_part, float *kp, float *kpt, int64_t ldt, void *stream);

/* tb_linear_kv_part_pool that also writes the smoothed K codes and scales
 * (_quantize_token_blocks of k - k_mean, attention.py:201-220, bit-identical
 * to tb_pool_quant_tokens(k, k_mean, kv_block)): k_codes int8 [H, L, d],
 * k_scales f32 [H, nkv], from the same K tiles (no separate K pass); needs
 * k_mean f32 [H, d] on the stream first.  k_codes / k_scales NULL = _pool. */
int tb_linear_kv_part_codes(const void *k, const void *v, int64_t H, int64_t L, int64_t d, int64_t kv_block,
                            int64_t dx, void *kv_part, float *kp, float *kpt, int64_t ldt, const float *k_mean,
                            int8_t *k_codes, float *k_scales, void *stream);

/* DiT glue in one pass: s = x (+ y) (+ alpha * emb[cols]) -> sum_out (f32,
 * optional, may alias x or y) and RMSNorm(s) * gain (layer_norm = 0) or
 * LayerNorm(s) * gain + offset (layer_norm = 1) as bf16 norm_out
 * (sampler.py:34-53 semantics, eps added inside the root). */
int tb_add_norm(const float *x, const float *y, const float *emb, float alpha, const float *gain, const float *offset,
                int64_t rows, int64_t cols, float eps, int layer_norm, float *sum_out, void *norm_out, void *stream);
/* tb_add_norm fused with tb_quantize_blockwise (block 128) of its bf16 norm
 * output -- the norm-fed activation quantizations of the DiT block (the
 * RMSNorm -> qkv and LayerNorm -> mlp_in operands, sampler.py:161,180 with
 * quantized_linear_forward's blockquant.py:174) in one HBM pass: q int8
 * [rows, cols], scales f32 [ceil(rows/128), cols/128], bit-identical to the
 * two calls.  cols % 128 == 0, cols <= 6144; sum_out optional. */
int tb_add_norm_quant(const float *x, const float *y, const float *emb, float alpha, const float *gain,
                      const float *offset, int64_t rows, int64_t cols, float eps, int layer_norm, float *sum_out,
                      int8_t *q, float *scales, void *stream);

/* Delta merge step (replaces the loop body of merge.apply_deltas,
 * merge.py:63-70): acc[i] = acc[i] + fl(c * x[i]) with two RN roundings, the
 * numpy order bit-for-bit; called once per delta in list order. */
int tb_axpy_rn(float *acc, const float *x, float c, int64_t n, void *stream);

/* quantize_blockwise (block 128) of a logical [rows, cols] matrix stored as
 * cols/128 planes [rows, 128] (a head-major attention output [H, L, 128]);
 * codes [rows, cols] row-major, scales [ceil(rows/128), cols/128]. */
int tb_quantize_blockwise_planar(const void *x, int dtype, int64_t rows, int64_t cols, int8_t *q, float *scales,
                                 void *stream);

/* tb_w8a8_gemm_fast with epilogue options for the DiT block:
 * plane > 0 (divides 128 and N, bf16 out): the output is stored as N/plane
 * planes [M, plane] -- the qkv projection lands head-major [3, H, M, head_dim];
 * act == 1: GELU (tanh form, sampler.py:55-58) applied to the result. */
int tb_w8a8_gemm_fast_ex(const int8_t *a, const float *sa, const int8_t *bt, const float *sb, const float *bias,
                         int64_t M, int64_t N, int64_t K, int64_t block, void *out, int out_dtype, int64_t plane,
                         int act, void *stream);

/* tb_w8a8_gemm_fast_ex (+ optional GELU) whose epilogue block-quantizes the
 * bf16-rounded result for the next projection (sampler.py:180-185:
 * mlp_in -> GELU -> quantize -> mlp_out): codes q_out [M, N] int8 and scales
 * [ceil(M/128), N/128], bit-identical to tb_quantize_blockwise of the bf16
 * tb_w8a8_gemm_fast_ex output.  Needs block 128, N % 256 == 0, M >= 256
 * (TB_EUNSUPPORTED otherwise: the caller runs the two-kernel path). */
int tb_w8a8_gemm_quant(const int8_t *a, const float *sa, const int8_t *bt, const float *sb, const float *bias,
                       int64_t M, int64_t N, int64_t K, int64_t block, int act, int8_t *q_out, float *scales_out,
                       void *stream);

/* Fused Ulysses forward exchange (new, multi-GPU; replaces the q/k/v
 * all-to-all after the qkv projection of toy_block_forward, sampler.py:
 * 161-170): fast-mode W8A8 of this rank's token shard (sequence rows [row0,
 * row0 + M)) whose epilogue TMA-stores every output box straight into the
 * head owner's buffer.  peers: HOST array of P (<= 8) device pointers (peer
 * memory from tb_peer_alloc / tb_peer_import), each bf16 [3*(H/P), L, 128] = the q,
 * k, v planes of that rank's heads over all L tokens.  N = 3*H*128; 2-SM
 * kernel shapes only (block 128, M >= 256), TB_EUNSUPPORTED otherwise. */
int tb_w8a8_gemm_qkv_peers(const int8_t *a, const float *sa, const int8_t *bt, const float *sb, const float *bias,
                           int64_t M, int64_t N, int64_t K, int64_t block, void *const *peers, int64_t P,
                           int64_t H, int64_t row0, int64_t L, void *stream);

/* Fast-mode W8A8: identical operands, the two block scales folded into one
 * FMA per element (tolerance-level, not bit-exact); used by the DiT step. */
int tb_w8a8_gemm_fast(const int8_t *a, const float *sa, const int8_t *bt, const float *sb,
                      const float *bias, int64_t M, int64_t N, int64_t K, int64_t block,
                      void *out, int out_dtype, void *stream);

/* ----------------------------------------------------------- DiT pieces */

/* sampler.rmsnorm / layernorm (sampler.py:34-52), f32 rows. */
int tb_rmsnorm(const float *x, const float *gain, int64_t rows, int64_t cols, float eps,
               float *out, void *stream);
int tb_layernorm(const float *x, const float *gain, const float *offset, int64_t rows,
                 int64_t cols, float eps, float *out, void *stream);
/* sampler._gelu tanh approximation (sampler.py:55-58), in place allowed. */
int tb_gelu(const float *x, int64_t n, float *out, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* TB_CAPI_H */

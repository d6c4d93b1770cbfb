/*
 * tb_oracle.c -- CPU restatement of the order-sensitive arithmetic on the
 * TurboDiffusion hot path (TEST INFRASTRUCTURE ONLY).
 *
 * This file is the checker, never the product: only tests/, the smoke()
 * entry point and bench.py's cpu_baseline / --impl reference legs may load
 * it.  The CUDA product path in paper_2512_16093_b200/ never links it.
 *
 * The reference (/root/reference/pkg/src/turbobench) is pure numpy; the
 * summation orders of its numpy/OpenBLAS reductions are third-party
 * behaviour (numpy 2.3.5 + scipy-openblas 0.3.30, SkylakeX kernel).  They
 * are restated here explicitly and pinned against golden vectors produced
 * by the reference itself (tests/golden/make_golden.py).
 *
 * Build: make -C oracle   (gcc -O2 -ffp-contract=off; fmaf is used only
 * where OpenBLAS uses an FMA chain).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* numpy pairwise summation (numpy/_core/src/umath/loops_utils.h.src,
 * pairwise_sum for FLOAT, PW_BLOCKSIZE 128) over n strided floats. */
static float pw_sum(const float *a, int64_t n, int64_t stride) {
    if (n < 8) {
        float res = -0.0f;
        for (int64_t i = 0; i < n; i++) res += a[i * stride];
        return res;
    } else if (n <= 128) {
        float r[8];
        for (int j = 0; j < 8; j++) r[j] = a[j * stride];
        int64_t i;
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += a[(i + j) * stride];
        float res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i * stride];
        return res;
    } else {
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        return pw_sum(a, n2, stride) + pw_sum(a + n2 * stride, n - n2, stride);
    }
}

/* pool_block_means, attention.py:256-266.  np.add.reduceat(x, starts, axis=1)
 * seeds each segment with its first row and adds the pairwise sum of the
 * remaining rows (FLOAT_add binary-reduce loop); the mean divides by the
 * f32 extent. */
void orc_pool_block_means(const float *x, int64_t H, int64_t L, int64_t d,
                          int64_t block, float *out) {
    int64_t nb = (L + block - 1) / block;
    for (int64_t h = 0; h < H; h++)
        for (int64_t b = 0; b < nb; b++) {
            int64_t lo = b * block;
            int64_t e = (lo + block < L ? block : L - lo);
            for (int64_t c = 0; c < d; c++) {
                const float *p = x + (h * L + lo) * d + c;
                float acc = p[0];
                if (e > 1) acc = acc + pw_sum(p + d, e - 1, d);
                out[(h * nb + b) * d + c] = acc / (float)e;
            }
        }
}

/* smooth_keys k_mean, attention.py:179-188: k.mean(axis=1) is a sequential
 * f32 chain over tokens (strided reduce), divided by f32(L). */
void orc_kmean(const float *k, int64_t H, int64_t L, int64_t d, float *kmean) {
    for (int64_t h = 0; h < H; h++)
        for (int64_t c = 0; c < d; c++) {
            float acc = 0.0f;
            const float *p = k + h * L * d + c;
            for (int64_t t = 0; t < L; t++) acc += p[t * d];
            kmean[h * d + c] = acc / (float)L;
        }
}

/* the shared quantization rule (attention.py:215-219, blockquant.py:105-109):
 * scale = f32(f64(absmax)/127) == am/127.f (RN; double rounding innocuous),
 * code = clip(rint(x / safe), -127, 127) with an IEEE f32 divide. */
static inline int8_t quant_code(float x, float safe) {
    float r = nearbyintf(x / safe);
    if (r > 127.f) r = 127.f;
    if (r < -127.f) r = -127.f;
    return (int8_t)r;
}

static inline float quant_scale(float am) { return (float)((double)am / 127.0); }

/* _quantize_token_blocks, attention.py:201-220 (x already centred for K). */
void orc_quant_token_blocks(const float *x, int64_t H, int64_t L, int64_t d,
                            int64_t block, int8_t *codes, float *scales) {
    int64_t nb = (L + block - 1) / block;
    for (int64_t h = 0; h < H; h++)
        for (int64_t b = 0; b < nb; b++) {
            int64_t lo = b * block, hi = lo + block < L ? lo + block : L;
            float am = 0.0f;
            for (int64_t t = lo; t < hi; t++)
                for (int64_t c = 0; c < d; c++) {
                    float a = fabsf(x[(h * L + t) * d + c]);
                    if (a > am) am = a;
                }
            float s = quant_scale(am);
            scales[h * nb + b] = s;
            float safe = (s == 0.0f) ? 1.0f : s;
            for (int64_t t = lo; t < hi; t++)
                for (int64_t c = 0; c < d; c++)
                    codes[(h * L + t) * d + c] = quant_code(x[(h * L + t) * d + c], safe);
        }
}

/* kc = k - k_mean (attention.py:188), then token-block quantization. */
void orc_quant_k(const float *k, const float *kmean, int64_t H, int64_t L, int64_t d,
                 int64_t block, float *kc, int8_t *codes, float *scales) {
    for (int64_t h = 0; h < H; h++)
        for (int64_t t = 0; t < L; t++)
            for (int64_t c = 0; c < d; c++)
                kc[(h * L + t) * d + c] = k[(h * L + t) * d + c] - kmean[h * d + c];
    orc_quant_token_blocks(kc, H, L, d, block, codes, scales);
}

/* block scores qp @ kp^T, attention.py:280 (numpy matmul -> cblas_sgemm,
 * which OpenBLAS sees as a TN product C^T = kp . qp^T).  Two SkylakeX paths:
 *  - the regular sgemm kernel: one FMA chain per output from 0 over the
 *    inner dimension (pinned at d=8..128, nq*nkv >= 4096);
 *  - the small-matrix TN kernel, taken when M*N <= 1200, K >= 32 and
 *    M*N*K <= 1e6: 16 lane accumulators (lane = t mod 16, FMA chains), then
 *    an adjacent-pair tree reduction of the 16 lanes.
 * Both pinned against reference golden vectors (tests/test_oracle_golden.py). */
static int small_tn_path(int64_t nq, int64_t nkv, int64_t d) {
    double mnk = (double)nq * (double)nkv * (double)d;
    return nq * nkv <= 1200 && d >= 32 && mnk <= 1e6;
}

void orc_block_scores(const float *qp, const float *kp, int64_t H, int64_t nq,
                      int64_t nkv, int64_t d, float *scores) {
    int small = small_tn_path(nq, nkv, d);
    for (int64_t h = 0; h < H; h++)
        for (int64_t i = 0; i < nq; i++)
            for (int64_t j = 0; j < nkv; j++) {
                const float *a = qp + (h * nq + i) * d;
                const float *b = kp + (h * nkv + j) * d;
                float acc = 0.0f;
                if (!small) {
                    for (int64_t t = 0; t < d; t++) acc = fmaf(a[t], b[t], acc);
                } else {
                    float lane[16] = {0};
                    for (int64_t t = 0; t < d; t++) lane[t % 16] = fmaf(a[t], b[t], lane[t % 16]);
                    for (int w = 8; w >= 1; w /= 2)
                        for (int l = 0; l < w; l++) lane[l] = lane[2 * l] + lane[2 * l + 1];
                    acc = lane[0];
                }
                scores[(h * nq + i) * nkv + j] = acc;
            }
}

typedef struct { float s; int64_t j; } scored_t;

static int cmp_desc(const void *pa, const void *pb) {
    const scored_t *a = (const scored_t *)pa, *b = (const scored_t *)pb;
    if (a->s > b->s) return -1;
    if (a->s < b->s) return 1;
    return (a->j < b->j) ? -1 : (a->j > b->j);   /* stable: low index wins ties */
}

static int cmp_i64(const void *pa, const void *pb) {
    int64_t a = *(const int64_t *)pa, b = *(const int64_t *)pb;
    return (a < b) ? -1 : (a > b);
}

/* select_topk_blocks, attention.py:269-284: argsort(-scores, stable)[:count]
 * then ascending sort.  numpy compares -0.0 == +0.0, as does cmp_desc. */
void orc_topk_from_scores(const float *scores, int64_t rows, int64_t nkv, int64_t count,
                          int64_t *idx) {
    scored_t *buf = (scored_t *)malloc(sizeof(scored_t) * (size_t)(nkv > 0 ? nkv : 1));
    for (int64_t r = 0; r < rows; r++) {
        for (int64_t j = 0; j < nkv; j++) { buf[j].s = scores[r * nkv + j]; buf[j].j = j; }
        qsort(buf, (size_t)nkv, sizeof(scored_t), cmp_desc);
        for (int64_t c = 0; c < count; c++) idx[r * count + c] = buf[c].j;
        qsort(idx + r * count, (size_t)count, sizeof(int64_t), cmp_i64);
    }
    free(buf);
}

void orc_topk(const float *qp, const float *kp, int64_t H, int64_t nq, int64_t nkv,
              int64_t d, int64_t count, int64_t *idx) {
    float *scores = (float *)malloc(sizeof(float) * (size_t)(H * nq * nkv + 1));
    orc_block_scores(qp, kp, H, nq, nkv, d, scores);
    orc_topk_from_scores(scores, H * nq, nkv, count, idx);
    free(scores);
}

/* quantize_blockwise, blockquant.py:91-110.  Returns -1 on non-finite input
 * (the reference raises ValueError, :103-104). */
int orc_quantize_blockwise(const float *m, int64_t rows, int64_t cols, int64_t block,
                           int8_t *q, float *scales) {
    for (int64_t i = 0; i < rows * cols; i++)
        if (!isfinite(m[i])) return -1;
    int64_t nr = (rows + block - 1) / block, nc = (cols + block - 1) / block;
    for (int64_t bi = 0; bi < nr; bi++)
        for (int64_t bj = 0; bj < nc; bj++) {
            int64_t r0 = bi * block, r1 = r0 + block < rows ? r0 + block : rows;
            int64_t c0 = bj * block, c1 = c0 + block < cols ? c0 + block : cols;
            float am = 0.0f;
            for (int64_t r = r0; r < r1; r++)
                for (int64_t c = c0; c < c1; c++) {
                    float a = fabsf(m[r * cols + c]);
                    if (a > am) am = a;
                }
            float s = quant_scale(am);
            scales[bi * nc + bj] = s;
            float safe = (s == 0.0f) ? 1.0f : s;
            for (int64_t r = r0; r < r1; r++)
                for (int64_t c = c0; c < c1; c++)
                    q[r * cols + c] = quant_code(m[r * cols + c], safe);
        }
    return 0;
}

/* w8a8_matmul, blockquant.py:132-161: per k-block an exact integer segment,
 * seg *= row_scale, seg *= col_scale, out += seg in ascending k-block order
 * starting from out = 0. */
void orc_w8a8(const int8_t *aq, const float *as, const int8_t *bq, const float *bs,
              int64_t M, int64_t K, int64_t N, int64_t block, float *out) {
    int64_t nkb = (K + block - 1) / block, nnb = (N + block - 1) / block;
    int64_t nmb = (M + block - 1) / block;
    (void)nmb;
    int64_t *seg = (int64_t *)malloc(sizeof(int64_t) * (size_t)(N > 0 ? N : 1));
    for (int64_t i = 0; i < M; i++) {
        float *o = out + i * N;
        for (int64_t j = 0; j < N; j++) o[j] = 0.0f;
        for (int64_t kb = 0; kb < nkb; kb++) {
            int64_t k0 = kb * block, k1 = k0 + block < K ? k0 + block : K;
            memset(seg, 0, sizeof(int64_t) * (size_t)N);
            for (int64_t k = k0; k < k1; k++) {
                int64_t a = aq[i * K + k];
                if (!a) continue;
                const int8_t *brow = bq + k * N;
                for (int64_t j = 0; j < N; j++) seg[j] += a * (int64_t)brow[j];
            }
            float rs = as[(i / block) * nkb + kb];
            for (int64_t j = 0; j < N; j++) {
                float v = (float)seg[j];
                v = v * rs;
                v = v * bs[kb * nnb + j / block];
                o[j] = o[j] + v;
            }
        }
    }
    free(seg);
}

/* feature map phi, attention.py:287-290. */
void orc_feature_map(const float *x, int64_t n, float *out) {
    for (int64_t i = 0; i < n; i++) out[i] = x[i] >= 0.0f ? x[i] + 1.0f : expf(x[i]);
}

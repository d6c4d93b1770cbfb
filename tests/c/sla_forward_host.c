/* A plain-C host of the library (no Python, no torch): reads bf16 q, k, v
 * [H, L, 128] from files, runs the whole sla_attention through the C ABI
 * (tb_sla_workspace_bytes + tb_sla_forward on its own CUDA stream) and writes
 * the f32 output.  Built and run by tests/test_gpu_c_host.py:
 *   gcc sla_forward_host.c -I include -I $CUDA/include -L pkg -ltb200 -L $CUDA/lib64 -lcudart
 * usage: sla_forward_host H L q_block q.bin k.bin v.bin out.bin */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <cuda_runtime.h>

#include "tb_capi.h"

static void *load(const char *path, size_t bytes) {
    FILE *f = fopen(path, "rb");
    if (!f) { perror(path); exit(2); }
    void *h = malloc(bytes);
    if (fread(h, 1, bytes, f) != bytes) { fprintf(stderr, "short read %s\n", path); exit(2); }
    fclose(f);
    void *d = NULL;
    if (cudaMalloc(&d, bytes) != cudaSuccess || cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice) != cudaSuccess) {
        fprintf(stderr, "cuda upload failed\n");
        exit(3);
    }
    free(h);
    return d;
}

int main(int argc, char **argv) {
    if (argc != 8) { fprintf(stderr, "usage: %s H L q_block q.bin k.bin v.bin out.bin\n", argv[0]); return 1; }
    const int64_t H = atoll(argv[1]), L = atoll(argv[2]), qb = atoll(argv[3]), d = 128;
    const size_t in_bytes = (size_t)(H * L * d) * 2, out_bytes = (size_t)(H * L * d) * 4;
    void *q = load(argv[4], in_bytes), *k = load(argv[5], in_bytes), *v = load(argv[6], in_bytes);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    const int64_t ws_bytes = tb_sla_workspace_bytes(H, L, d, qb, 64, 0.1, 1.0f, TB_BF16);
    if (ws_bytes < 0) { fprintf(stderr, "workspace query: %s\n", tb_last_error()); return 4; }
    void *ws = NULL, *out = NULL;
    cudaMalloc(&ws, (size_t)ws_bytes);
    cudaMalloc(&out, out_bytes);
    const int rc = tb_sla_forward(q, k, v, TB_BF16, H, L, d, qb, 64, 0.1, 1.0f, 1.0f / sqrtf((float)d), ws, ws_bytes,
                                  out, TB_F32, (void *)st);
    if (rc != TB_OK) { fprintf(stderr, "tb_sla_forward: %d %s\n", rc, tb_last_error()); return 5; }
    if (cudaStreamSynchronize(st) != cudaSuccess) { fprintf(stderr, "stream sync failed\n"); return 6; }
    float *h = (float *)malloc(out_bytes);
    cudaMemcpy(h, out, out_bytes, cudaMemcpyDeviceToHost);
    FILE *f = fopen(argv[7], "wb");
    fwrite(h, 1, out_bytes, f);
    fclose(f);
    printf("ok workspace=%lld\n", (long long)ws_bytes);
    return 0;
}

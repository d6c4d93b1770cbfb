// ring_upload.cu -- host-memory experiment for the drop-in's upload (tools only).
// Uploads N f32 values as bf16 (upper halves) to the device two ways, 16 threads:
//  big:  threads narrow into one big pinned buffer with non-temporal stores, the
//        DMA follows in 64 MB pieces (what the pipeline does today, roughly)
//  ring: each thread narrows a SLOT-sized piece into one of its own two small pinned
//        slots with ordinary (cached) stores and immediately issues the DMA of that
//        piece, so the copy engine reads the lines while they are still in cache
// build: nvcc -O3 -Xcompiler -mavx2 -o gpurun_out/ring_upload tools/ring_upload.cu -lpthread
#include <cuda_runtime.h>
#include <immintrin.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

static void narrow(uint16_t *dst, const float *src, int64_t n, bool nt) {
    const uint32_t *u = (const uint32_t *)src;
    int64_t i = 0;
    for (; i + 16 <= n; i += 16) {
        __m256i a = _mm256_loadu_si256((const __m256i *)(u + i)), b = _mm256_loadu_si256((const __m256i *)(u + i + 8));
        __m256i pk = _mm256_permute4x64_epi64(_mm256_packus_epi32(_mm256_srli_epi32(a, 16), _mm256_srli_epi32(b, 16)), 0xD8);
        if (nt) _mm256_stream_si256((__m256i *)(dst + i), pk);
        else _mm256_store_si256((__m256i *)(dst + i), pk);
    }
    for (; i < n; i++) dst[i] = (uint16_t)(u[i] >> 16);
    if (nt) _mm_sfence();
}

int main(int argc, char **argv) {
    const int T = argc > 1 ? atoi(argv[1]) : 16;
    const int64_t N = (int64_t)1161216000;                 // cfg4 q + k + v elements
    const int64_t slot_elems = argc > 2 ? atoll(argv[2]) : (1 << 19);
    std::vector<float> srcv(N);
    for (int64_t i = 0; i < N; i += 1) ((uint32_t *)srcv.data())[i] = (uint32_t)((i * 2654435761u) & 0xFFFF0000u);
    const float *src = srcv.data();
    uint16_t *dev;
    cudaMalloc(&dev, N * 2);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    // ---- big: staging buffer of 256 MB pieces (double-buffered), NT stores, one DMA per piece
    {
        const int64_t piece = 128ll << 20;                      // elements per piece
        uint16_t *buf[2];
        cudaHostAlloc(&buf[0], piece * 2, cudaHostAllocPortable);
        cudaHostAlloc(&buf[1], piece * 2, cudaHostAllocPortable);
        cudaEvent_t ev[2];
        cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming);
        for (int rep = 0; rep < 3; rep++) {
            double t0 = now();
            for (int64_t p = 0, k = 0; p < N; p += piece, k++) {
                const int s = (int)(k & 1);
                if (k >= 2) cudaEventSynchronize(ev[s]);
                const int64_t m = std::min(piece, N - p);
                std::vector<std::thread> th;
                for (int t = 0; t < T; t++)
                    th.emplace_back([&, t] {
                        const int64_t a = m * t / T, z = m * (t + 1) / T;
                        narrow(buf[s] + a, src + p + a, z - a, true);
                    });
                for (auto &x : th) x.join();
                cudaMemcpyAsync(dev + p, buf[s], m * 2, cudaMemcpyHostToDevice, st);
                cudaEventRecord(ev[s], st);
            }
            cudaStreamSynchronize(st);
            double t1 = now();
            printf("big NT staging + DMA: %.1f ms (%.1f GB/s of wire bytes)\n", (t1 - t0) * 1e3, N * 2 / (t1 - t0) / 1e9);
        }
        cudaFreeHost(buf[0]);
        cudaFreeHost(buf[1]);
    }
    // ---- ring: per-thread 2 slots, cached stores, DMA per slot
    for (int nt = 0; nt < 2; nt++) {
        std::vector<uint16_t *> slots(2 * T);
        std::vector<cudaEvent_t> evs(2 * T);
        for (int i = 0; i < 2 * T; i++) {
            cudaHostAlloc(&slots[i], slot_elems * 2, cudaHostAllocPortable);
            cudaEventCreateWithFlags(&evs[i], cudaEventDisableTiming);
        }
        const int64_t npieces = (N + slot_elems - 1) / slot_elems;
        for (int rep = 0; rep < 3; rep++) {
            std::atomic<int64_t> next{0};
            double t0 = now();
            std::vector<std::thread> th;
            for (int t = 0; t < T; t++)
                th.emplace_back([&, t] {
                    int64_t used = 0;
                    for (;;) {
                        const int64_t p = next.fetch_add(1);
                        if (p >= npieces) break;
                        const int s = 2 * t + (int)(used & 1);
                        if (used >= 2) cudaEventSynchronize(evs[s]);
                        used++;
                        const int64_t a = p * slot_elems, m = std::min(slot_elems, N - a);
                        narrow(slots[s], src + a, m, nt == 1);
                        cudaMemcpyAsync(dev + a, slots[s], m * 2, cudaMemcpyHostToDevice, st);
                        cudaEventRecord(evs[s], st);
                    }
                });
            for (auto &x : th) x.join();
            cudaStreamSynchronize(st);
            double t1 = now();
            printf("ring %s stores, slot %lld KB: %.1f ms (%.1f GB/s of wire bytes)\n", nt ? "NT" : "cached",
                   (long long)(slot_elems * 2 / 1024), (t1 - t0) * 1e3, N * 2 / (t1 - t0) / 1e9);
        }
        for (int i = 0; i < 2 * T; i++) cudaFreeHost(slots[i]);
    }
    // pure DMA from one pinned buffer (the PCIe bound)
    {
        uint16_t *h;
        const int64_t m = 256ll << 20;
        cudaHostAlloc(&h, m * 2, 0);
        memset(h, 1, m * 2);
        double t0 = now();
        for (int64_t p = 0; p + m <= N; p += m) cudaMemcpyAsync(dev + p, h, m * 2, cudaMemcpyHostToDevice, st);
        cudaStreamSynchronize(st);
        double t1 = now();
        printf("DMA only (pinned, %lld MB copies): %.1f GB/s\n", (long long)(m * 2 >> 20), (N / m) * m * 2 / (t1 - t0) / 1e9);
    }
    return 0;
}

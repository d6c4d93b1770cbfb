// peer.cu -- NVLink peer memory for the fused Ulysses exchanges (SURVEY.md §8
// e1): dedicated allocations exported / imported with CUDA IPC handles (one
// process per GPU; also valid for two processes sharing one GPU, which is how
// the multi-rank path is tested on a one-GPU box), and a stream-ordered
// device barrier over per-rank flag blocks in that memory.
//
// Barrier protocol: each rank owns a flag block of P uint32 slots; barrier
// number e (monotonic per group) has rank r store e into slot r of every
// peer's block with release semantics at system scope (after a system-scope
// fence, so the stores of the kernels that precede it on the stream are
// visible first), then spin with acquire loads until every slot of its own
// block has reached e.  The kernels after it on the stream therefore see
// every peer's stores issued before that peer's barrier.
#include <cstring>

#include "common.cuh"

namespace tb {

__global__ void peer_barrier_kernel(uint32_t *const *__restrict__ flags, int P, int rank, uint32_t epoch) {
    if (threadIdx.x == 0) asm volatile("fence.acq_rel.sys;" ::: "memory");
    __syncwarp();
    const int r = threadIdx.x;
    if (r < P) {
        uint32_t *dst = flags[r] + rank;            // my slot in rank r's block
        asm volatile("st.release.sys.global.u32 [%0], %1;" :: "l"(dst), "r"(epoch) : "memory");
        const uint32_t *mine = flags[rank] + r;     // rank r's slot in my block
        uint32_t v;
        do {
            asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(mine) : "memory");
        } while ((int32_t)(v - epoch) < 0);
    }
    __syncwarp();
    if (threadIdx.x == 0) asm volatile("fence.acq_rel.sys;" ::: "memory");
}

}  // namespace tb

using namespace tb;

extern "C" int tb_peer_alloc(int64_t bytes, void **ptr) {
    TB_REQUIRE(ptr != nullptr && bytes > 0, "bad allocation request");
    *ptr = nullptr;
    if (cudaMalloc(ptr, (size_t)bytes) != cudaSuccess) return fail(TB_ECUDA, "cudaMalloc (peer buffer) failed");
    // zeroed (barrier flags start at epoch 0) and complete before the handle
    // can reach a peer
    if (cudaMemset(*ptr, 0, (size_t)bytes) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess)
        return fail(TB_ECUDA, "cudaMemset (peer buffer) failed");
    return TB_OK;
}

extern "C" int tb_peer_free(void *ptr) {
    if (ptr && cudaFree(ptr) != cudaSuccess) return fail(TB_ECUDA, "cudaFree (peer buffer) failed");
    return TB_OK;
}

// handle: 64 bytes (cudaIpcMemHandle_t) for a tb_peer_alloc pointer
extern "C" int tb_peer_export(void *ptr, void *handle) {
    TB_REQUIRE(ptr != nullptr && handle != nullptr, "null pointer");
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, ptr) != cudaSuccess) return fail(TB_ECUDA, "cudaIpcGetMemHandle failed");
    memcpy(handle, &h, sizeof(h));
    return TB_OK;
}

extern "C" int tb_peer_import(const void *handle, void **ptr) {
    TB_REQUIRE(ptr != nullptr && handle != nullptr, "null pointer");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    if (cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
        return fail(TB_ECUDA, "cudaIpcOpenMemHandle failed");
    return TB_OK;
}

extern "C" int tb_peer_close(void *ptr) {
    if (ptr && cudaIpcCloseMemHandle(ptr) != cudaSuccess) return fail(TB_ECUDA, "cudaIpcCloseMemHandle failed");
    return TB_OK;
}

// flags: DEVICE array of P pointers to the ranks' flag blocks (P uint32 each)
extern "C" int tb_peer_barrier(uint32_t *const *flags, int64_t P, int64_t rank, uint32_t epoch, void *stream) {
    TB_REQUIRE(flags != nullptr && P >= 1 && P <= 32 && rank >= 0 && rank < P, "bad barrier group");
    peer_barrier_kernel<<<1, 32, 0, as_stream(stream)>>>(flags, (int)P, (int)rank, epoch);
    return check_launch("peer_barrier");
}

// ulysses.cu -- the Ulysses head-parallel exchange as C-ABI entry points
// (token shard [L/P, H, d] <-> head shard [H/P, L, d],
// one all-to-all each way over NCCL), for hosts that drive the hot path
// through the C ABI instead of torch.distributed.
//
// Layout (ulysses.py is the Python mirror; the tests check one against the
// other): rank r owns tokens [r*per, min((r+1)*per, L)) with per = ceil(L/P)
// rounded up to `align`, and heads [r*hp, (r+1)*hp) with hp = H/P.  Send and
// receive buffers are [P, per, hp, d]: for seq -> heads chunk j of the send
// buffer holds my tokens of head group j, chunk i of the receive buffer rank
// i's tokens of my heads (read as [P*per, hp, d] it is already the global
// token order); heads -> seq is the mirror image.  Rows past a shard's end are
// never read.  The exchange is one grouped ncclSend/ncclRecv per peer of a
// contiguous per*hp*d chunk; pack and unpack are one vectorised permute each.
//
// NCCL is resolved at run time (dlopen of libnccl.so.2 -- already mapped when
// torch is loaded), so libtb200.so has no link-time NCCL dependency; the
// communicator is the caller's (its ncclComm_t passed as void*), or one made
// with tb_nccl_unique_id / tb_nccl_comm_init.
#include <dlfcn.h>
#include <cstring>
#include <mutex>

#include "common.cuh"

namespace tb {
namespace {

// dst(i0, i1, i2) = src(i0, i1, i2) over rows of row_bytes (multiple of 16),
// with independent byte strides on both sides; rows whose sequence position
// pos0 + i0*pos_s0 + i1 is >= lim are skipped (past the end of the sequence).
__global__ void permute3_kernel(const uint8_t *__restrict__ src, uint8_t *__restrict__ dst, int64_t n0, int64_t n1,
                                int64_t n2, int64_t row_bytes, int64_t s0, int64_t s1, int64_t s2, int64_t d0,
                                int64_t d1, int64_t d2, int64_t pos0, int64_t pos_s0, int64_t lim) {
    const int64_t nv = row_bytes >> 4;
    const int64_t total = n0 * n1 * n2 * nv;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = idx % nv;
        int64_t r = idx / nv;
        const int64_t i2 = r % n2;
        r /= n2;
        const int64_t i1 = r % n1;
        const int64_t i0 = r / n1;
        if (pos0 + i0 * pos_s0 + i1 >= lim) continue;
        const uint4 w = *reinterpret_cast<const uint4 *>(src + i0 * s0 + i1 * s1 + i2 * s2 + v * 16);
        *reinterpret_cast<uint4 *>(dst + i0 * d0 + i1 * d1 + i2 * d2 + v * 16) = w;
    }
}

int permute3(const void *src, void *dst, int64_t n0, int64_t n1, int64_t n2, int64_t row_bytes, int64_t s0,
             int64_t s1, int64_t s2, int64_t d0, int64_t d1, int64_t d2, int64_t pos0, int64_t pos_s0, int64_t lim,
             cudaStream_t st) {
    const int64_t total = n0 * n1 * n2 * (row_bytes >> 4);
    if (total == 0) return TB_OK;
    const int64_t blocks = imin64(cdiv(total, 256), 148 * 16);
    permute3_kernel<<<(unsigned)blocks, 256, 0, st>>>((const uint8_t *)src, (uint8_t *)dst, n0, n1, n2, row_bytes,
                                                      s0, s1, s2, d0, d1, d2, pos0, pos_s0, lim);
    return check_launch("ulysses_permute");
}

// ------------------------------------------------------------- NCCL (dlopen)
struct NcclUid { char b[128]; };                 // ncclUniqueId (NCCL_UNIQUE_ID_BYTES)
constexpr int NCCL_UINT8 = 1;                    // ncclDataType_t ncclUint8
struct NcclApi {
    int (*get_unique_id)(NcclUid *) = nullptr;
    int (*comm_init_rank)(void **, int, NcclUid, int) = nullptr;
    int (*comm_destroy)(void *) = nullptr;
    int (*group_start)() = nullptr;
    int (*group_end)() = nullptr;
    int (*send)(const void *, size_t, int, int, void *, cudaStream_t) = nullptr;
    int (*recv)(void *, size_t, int, int, void *, cudaStream_t) = nullptr;
    const char *(*error_string)(int) = nullptr;
    bool ok = false;
};

const NcclApi &nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        api.group_start = reinterpret_cast<decltype(api.group_start)>(dlsym(h, "ncclGroupStart"));
        api.group_end = reinterpret_cast<decltype(api.group_end)>(dlsym(h, "ncclGroupEnd"));
        api.send = reinterpret_cast<decltype(api.send)>(dlsym(h, "ncclSend"));
        api.recv = reinterpret_cast<decltype(api.recv)>(dlsym(h, "ncclRecv"));
        api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
        api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.group_start && api.group_end &&
                 api.send && api.recv;
    });
    return api;
}

int nccl_fail(const char *what, int rc) {
    const NcclApi &n = nccl();
    return fail(TB_ECUDA, std::string(what) + ": " + (n.error_string ? n.error_string(rc) : "nccl error"));
}

// one grouped send/recv per peer of `chunk` bytes (P == 1: a device copy)
int exchange(const void *send, void *recv, int64_t P, int64_t chunk, void *comm, cudaStream_t st) {
    if (P == 1) {
        if (cudaMemcpyAsync(recv, send, (size_t)chunk, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
            return fail(TB_ECUDA, "ulysses: self copy failed");
        return TB_OK;
    }
    const NcclApi &n = nccl();
    if (!n.ok) return fail(TB_ECUDA, "ulysses: libnccl.so.2 not loadable");
    int rc = n.group_start();
    if (rc) return nccl_fail("ncclGroupStart", rc);
    for (int64_t j = 0; j < P; j++) {
        rc = n.send(static_cast<const uint8_t *>(send) + j * chunk, (size_t)chunk, NCCL_UINT8, (int)j, comm, st);
        if (rc) break;
        rc = n.recv(static_cast<uint8_t *>(recv) + j * chunk, (size_t)chunk, NCCL_UINT8, (int)j, comm, st);
        if (rc) break;
    }
    const int rc2 = n.group_end();
    if (rc) return nccl_fail("ncclSend/ncclRecv", rc);
    if (rc2) return nccl_fail("ncclGroupEnd", rc2);
    return TB_OK;
}

}  // namespace
}  // namespace tb

using namespace tb;

extern "C" int64_t tb_ulysses_shard(int64_t L, int64_t P, int64_t align) {
    if (P < 1 || align < 1) return -1;
    const int64_t per = cdiv(L, P);
    return cdiv(per, align) * align;
}

extern "C" int64_t tb_ulysses_workspace_bytes(int64_t L, int64_t H, int64_t d, int64_t esize, int64_t P,
                                              int64_t align) {
    if (P < 1 || H % P) return -1;
    return P * tb_ulysses_shard(L, P, align) * (H / P) * d * esize;       // one of the two buffers
}

extern "C" int tb_ulysses_seq_to_heads(const void *x, int64_t L, int64_t H, int64_t d, int64_t esize, int64_t P,
                                       int64_t rank, int64_t align, void *send_ws, void *recv_ws, void *out,
                                       void *comm, int stages, void *stream) {
    TB_REQUIRE(P >= 1 && rank >= 0 && rank < P && H % P == 0, "need 0 <= rank < P and H % P == 0");
    TB_REQUIRE((d * esize) % 16 == 0, "head_dim * element size must be a multiple of 16 bytes");
    TB_REQUIRE(send_ws && recv_ws && (out || L == 0), "null buffer");
    TB_REQUIRE(!(stages & TB_UL_EXCHANGE) || P == 1 || comm != nullptr, "the exchange needs an NCCL communicator");
    cudaStream_t st = as_stream(stream);
    const int64_t per = tb_ulysses_shard(L, P, align), hp = H / P, rb = d * esize;
    const int64_t lo = imin64(rank * per, L), Lp = imin64(lo + per, L) - lo;
    TB_REQUIRE(x || Lp == 0, "null token shard");
    // pack: send[j, t, hh] = x[t, j*hp + hh]   (t < Lp)
    int rc = TB_OK;
    if (stages & TB_UL_PACK)
        rc = permute3(x, send_ws, P, Lp, hp, rb, hp * rb, H * rb, rb, per * hp * rb, hp * rb, rb, 0, 0, INT64_MAX, st);
    if (!rc && (stages & TB_UL_EXCHANGE)) rc = exchange(send_ws, recv_ws, P, per * hp * rb, comm, st);
    // unpack: out[hh, i*per + t] = recv[i, t, hh]   (i*per + t < L)
    if (!rc && (stages & TB_UL_UNPACK))
        rc = permute3(recv_ws, out, P, per, hp, rb, per * hp * rb, hp * rb, rb, per * rb, rb, L * rb, 0, per, L, st);
    return rc;
}

extern "C" int tb_ulysses_heads_to_seq(const void *o, int64_t L, int64_t H, int64_t d, int64_t esize, int64_t P,
                                       int64_t rank, int64_t align, void *send_ws, void *recv_ws, void *out,
                                       void *comm, int stages, void *stream) {
    TB_REQUIRE(P >= 1 && rank >= 0 && rank < P && H % P == 0, "need 0 <= rank < P and H % P == 0");
    TB_REQUIRE((d * esize) % 16 == 0, "head_dim * element size must be a multiple of 16 bytes");
    TB_REQUIRE(send_ws && recv_ws && (o || L == 0), "null buffer");
    TB_REQUIRE(!(stages & TB_UL_EXCHANGE) || P == 1 || comm != nullptr, "the exchange needs an NCCL communicator");
    cudaStream_t st = as_stream(stream);
    const int64_t per = tb_ulysses_shard(L, P, align), hp = H / P, rb = d * esize;
    const int64_t lo = imin64(rank * per, L), Lp = imin64(lo + per, L) - lo;
    TB_REQUIRE(out || Lp == 0, "null token-shard output");
    // pack: send[i, t, hh] = o[hh, i*per + t]   (i*per + t < L)
    int rc = TB_OK;
    if (stages & TB_UL_PACK)
        rc = permute3(o, send_ws, P, per, hp, rb, per * rb, rb, L * rb, per * hp * rb, hp * rb, rb, 0, per, L, st);
    if (!rc && (stages & TB_UL_EXCHANGE)) rc = exchange(send_ws, recv_ws, P, per * hp * rb, comm, st);
    // unpack: out[t, j*hp + hh] = recv[j, t, hh]   (t < Lp)
    if (!rc && (stages & TB_UL_UNPACK))
        rc = permute3(recv_ws, out, P, Lp, hp, rb, per * hp * rb, hp * rb, rb, hp * rb, H * rb, rb, 0, 0, INT64_MAX, st);
    return rc;
}

extern "C" int tb_nccl_unique_id(void *id128) {
    const NcclApi &n = nccl();
    TB_REQUIRE(id128 != nullptr, "null id buffer");
    if (!n.ok) return fail(TB_ECUDA, "libnccl.so.2 not loadable");
    NcclUid u;
    const int rc = n.get_unique_id(&u);
    if (rc) return nccl_fail("ncclGetUniqueId", rc);
    memcpy(id128, &u, sizeof(u));
    return TB_OK;
}

extern "C" int tb_nccl_comm_init(void **comm, const void *id128, int64_t nranks, int64_t rank) {
    const NcclApi &n = nccl();
    TB_REQUIRE(comm && id128 && nranks >= 1 && rank >= 0 && rank < nranks, "bad communicator arguments");
    if (!n.ok) return fail(TB_ECUDA, "libnccl.so.2 not loadable");
    NcclUid u;
    memcpy(&u, id128, sizeof(u));
    const int rc = n.comm_init_rank(comm, (int)nranks, u, (int)rank);
    return rc ? nccl_fail("ncclCommInitRank", rc) : TB_OK;
}

extern "C" int tb_nccl_comm_destroy(void *comm) {
    const NcclApi &n = nccl();
    if (!comm) return TB_OK;
    if (!n.ok) return fail(TB_ECUDA, "libnccl.so.2 not loadable");
    const int rc = n.comm_destroy(comm);
    return rc ? nccl_fail("ncclCommDestroy", rc) : TB_OK;
}

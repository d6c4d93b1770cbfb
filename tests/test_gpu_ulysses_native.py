"""The C-ABI Ulysses exchange (csrc/ulysses.cu) against the
Python/torch.distributed mirror's layout: one process, P = 1 through the full
op, and P = 2 / 4 / 8 emulated (each rank's pack, the all-to-all done as
chunk copies between the emulated ranks' buffers, each rank's unpack) --
bit-identical to slicing the global tensor, uneven and 128-aligned shards,
bf16 / int8 / f32 payloads."""
import pytest
import torch

from paper_2512_16093_b200 import ulysses as U

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2512_16093_b200 import _lib
    _lib.load(require_device=True)


def test_single_rank_full_op():
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn((300, 4, 128), generator=g, device="cuda").to(torch.bfloat16)
    out, _, _ = U.native_seq_to_heads(x, 300, 1, 0)
    assert torch.equal(out, x.permute(1, 0, 2))
    back, _, _ = U.native_heads_to_seq(out, 300, 1, 0)
    assert torch.equal(back, x)


@pytest.mark.parametrize("P,L,align", [(2, 1000, 1), (4, 1001, 1), (4, 1000, 128), (8, 4099, 128)])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.int8, torch.float32])
def test_emulated_ranks_match_global_layout(P, L, align, dtype):
    H, d = 8, 128
    g = torch.Generator(device="cuda").manual_seed(P * 100 + L)
    full = (torch.randn((L, H, d), generator=g, device="cuda") * 50).to(dtype)
    bounds = [U.token_bounds(L, P, r, align) for r in range(P)]
    # seq -> heads: pack on every rank, exchange by chunk copies, unpack
    sends, recvs = [], []
    for r in range(P):
        lo, hi = bounds[r]
        _, s, rv = U.native_seq_to_heads(full[lo:hi].contiguous(), L, P, r, align, stages=U.TB_UL_PACK)
        sends.append(s)
        recvs.append(rv)
    for r in range(P):
        for i in range(P):
            recvs[r][i].copy_(sends[i][r])
    hp = H // P
    heads = []
    for r in range(P):
        lo, hi = bounds[r]
        out, _, _ = U.native_seq_to_heads(full[lo:hi].contiguous(), L, P, r, align, stages=U.TB_UL_UNPACK,
                                          send=sends[r], recv=recvs[r])
        assert torch.equal(out, full[:, r * hp:(r + 1) * hp].permute(1, 0, 2)), r
        heads.append(out)
    # heads -> seq
    sends, recvs = [], []
    for r in range(P):
        _, s, rv = U.native_heads_to_seq(heads[r], L, P, r, align, stages=U.TB_UL_PACK)
        sends.append(s)
        recvs.append(rv)
    for r in range(P):
        for j in range(P):
            recvs[r][j].copy_(sends[j][r])
    for r in range(P):
        lo, hi = bounds[r]
        out, _, _ = U.native_heads_to_seq(heads[r], L, P, r, align, stages=U.TB_UL_UNPACK, send=sends[r],
                                          recv=recvs[r])
        assert torch.equal(out, full[lo:hi]), r


def test_exchange_needs_communicator():
    x = torch.zeros((64, 4, 128), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ValueError):
        U.native_seq_to_heads(x, 128, 2, 0)


def test_nccl_comm_through_the_c_abi(tmp_path):
    """tb_nccl_unique_id / tb_nccl_comm_init / tb_nccl_comm_destroy (libnccl.so.2
    resolved at run time) in a one-rank group."""
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"file://{tmp_path}/pg", rank=0, world_size=1)
    try:
        c = U.NcclComm()
        assert c.handle
        c.close()
    finally:
        dist.destroy_process_group()

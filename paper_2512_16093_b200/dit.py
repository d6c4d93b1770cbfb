"""Device-resident toy DiT + rCM few-step sampler (the cfg5 throughput path).

Same block as ``sampler.toy_block_forward`` (/root/reference/pkg/src/turbobench/
sampler.py:132-186): x + sigma*emb -> RMSNorm -> W8A8 qkv -> SLA attention ->
W8A8 out_proj -> residual -> LayerNorm -> W8A8 mlp_in -> GELU(tanh) -> W8A8
mlp_out -> residual, and the multistep consistency loop of sampler.py:281-302.
Differences from the drop-in ``sampler`` module are throughput choices only:
weights live on the device as transposed INT8 codes (the GEMM's K-major B
operand) with 128x128 scales, the projections use the single-FMA promotion,
and intermediate activations are bf16 (the residual stream stays f32).

Sequence parallel with Ulysses attention when torch.distributed is
initialised: each rank holds a token shard of x, weights are replicated, and
attention exchanges q/k/v/o with one all-to-all each way (ulysses.py).
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import ops, ulysses


@dataclass
class DeviceLinear:
    bt: torch.Tensor        # int8 [N, K] (transposed codes)
    scales: torch.Tensor    # f32 [K/128, N/128]

    @property
    def shape(self):
        return self.bt.shape[1], self.bt.shape[0]


@dataclass
class DeviceLayer:
    rms_gain: torch.Tensor
    ln_gain: torch.Tensor
    ln_offset: torch.Tensor
    sigma_emb: torch.Tensor
    qkv: DeviceLinear
    out_proj: DeviceLinear
    mlp_in: DeviceLinear
    mlp_out: DeviceLinear



# token-shard alignment of the sequence-parallel DiT (ulysses.token_bounds align):
# the 128-token quantization blocks of the attention output never straddle ranks
TOKEN_ALIGN = 128

def quantize_device_weight(w: torch.Tensor, block: int = 128) -> DeviceLinear:
    """blockquant.quantize_blockwise on device (bit-exact codes), stored transposed."""
    q, s = ops.quantize_blockwise(w, block, check_finite=False)
    return DeviceLinear(ops.transpose_codes(q), s)


def from_toy_layers(layers) -> list[DeviceLayer]:
    """ToyBlockWeights (f32 or BlockQuantized matrices) -> device layers."""
    from .blockquant import BlockQuantized

    def lin(m):
        if isinstance(m, BlockQuantized):
            return DeviceLinear(m.device_codes_t(), m.device_scales())
        t = m if isinstance(m, torch.Tensor) else torch.from_numpy(m)
        return quantize_device_weight(t.cuda().float())

    def vec(v):
        return (v if isinstance(v, torch.Tensor) else torch.from_numpy(v)).cuda().float().contiguous()

    return [DeviceLayer(vec(w.rms_gain), vec(w.ln_gain), vec(w.ln_offset), vec(w.sigma_emb), lin(w.qkv),
                        lin(w.out_proj), lin(w.mlp_in), lin(w.mlp_out)) for w in layers]


def random_layers(model_dim: int, ffn: int, num_layers: int, seed: int = 0) -> list[DeviceLayer]:
    """Random-init Wan-shaped toy DiT on device: N(0,1)/sqrt(fan_in) matrices
    (sampler.py:244-246), block-quantized by the device quantizer."""
    g = torch.Generator(device="cuda").manual_seed(seed)

    def mat(rows, cols):
        w = torch.randn((rows, cols), generator=g, device="cuda") / math.sqrt(rows)
        lin = quantize_device_weight(w)
        del w
        return lin

    def vec(scale, offset=0.0):
        return torch.randn(model_dim, generator=g, device="cuda") * scale + offset

    return [DeviceLayer(vec(0.1, 1.0), vec(0.1, 1.0), vec(0.1), vec(0.01), mat(model_dim, 3 * model_dim),
                        mat(model_dim, model_dim), mat(model_dim, ffn), mat(ffn, model_dim))
            for _ in range(num_layers)]


def _linear(x: torch.Tensor, w: DeviceLinear, out_dtype=torch.bfloat16) -> torch.Tensor:
    return ops.quantized_linear(x, w.bt, w.scales, 128, None, out_dtype, exact=False)


def block_forward(x: torch.Tensor, sigma: float, w: DeviceLayer, heads: int, sla: dict, L_global: int,
                  group=None, pending: torch.Tensor | None = None):
    """One block over the local token shard x [L_p, model_dim] (f32 residual stream).

    Returns (x2, p2): the block output is x2 + p2 -- the last residual add is
    left to the next block's fused add+norm (or to ``model_forward``)."""
    Lp, dim = x.shape
    hd = dim // heads
    # x1 = x (+ pending residual) + sigma*emb and the block-quantized RMSNorm(x1)
    # (the qkv projection's A operand).  Default: tb_add_norm + the blockwise
    # quantizer, two streaming passes (1.23 / 1.39 ms at cfg5); the one-pass
    # clustered tb_add_norm_quant (bit-identical) moves fewer
    # bytes but serialises its band phases at one CTA per SM (2.37 / 2.86 ms,
    # tools/time_add_norm.py), so it is opt-in: TB_DIT_FUSED_NORM_QUANT=1
    fused_nq = os.environ.get("TB_DIT_FUSED_NORM_QUANT") == "1" and ops.add_norm_quant_ok(dim)
    if fused_nq:
        x1, aq, asc = ops.add_norm_quant(x, pending, w.sigma_emb, float(sigma), w.rms_gain)
    else:
        x1, a = ops.add_norm(x, pending, w.sigma_emb, float(sigma), w.rms_gain)

    def attn(qh, kh, vh):
        return ops.sla_attention(qh, kh, vh, sla["q_block"], sla["kv_block"], sla["topk_ratio"],
                                 sla.get("linear_mix", 1.0), True, out_dtype=torch.bfloat16)

    if not fused_nq:
        aq, asc = ops.quantize_blockwise(a, 128, check_finite=False)
    multi = dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1
    if multi and hd == 128 and os.environ.get("TB_ULYSSES_P2P") == "1":
        # both exchanges fused into their producers over peer memory: the qkv
        # GEMM epilogue stores into the head owners' buffers, the attention
        # epilogue stores the int8 out-projection operand into the token owners'
        qh, kh, vh = ulysses.qkv_to_heads_p2p(aq, asc, w.qkv.bt, w.qkv.scales, L_global, heads, group, TOKEN_ALIGN)

        def attn_peer(qh_, kh_, vh_, peer_out):
            return ops.sla_attention(qh_, kh_, vh_, sla["q_block"], sla["kv_block"], sla["topk_ratio"],
                                     sla.get("linear_mix", 1.0), True, out_dtype=torch.int8,
                                     pv_fp8=sla.get("pv_fp8", False), peer_out=peer_out)
        oq, osc = ulysses.attn_return_p2p(qh, kh, vh, L_global, attn_peer, group, TOKEN_ALIGN)
    elif multi:
        # token shards are TOKEN_ALIGN-aligned (token_bounds(L, P, rank, TOKEN_ALIGN)),
        # so every 128x128 quantization block of the attention output is rank-local
        qkv = ops.w8a8_gemm(aq, asc, w.qkv.bt, w.qkv.scales, 128, None, torch.bfloat16, exact=False)
        q, k, v = (t.view(Lp, heads, hd).contiguous() for t in qkv.split(dim, dim=1))
        if hd == 128:
            def attn_q8(qh, kh, vh):
                return ops.sla_attention(qh, kh, vh, sla["q_block"], sla["kv_block"], sla["topk_ratio"],
                                         sla.get("linear_mix", 1.0), True, out_dtype=torch.int8,
                                         pv_fp8=sla.get("pv_fp8", False))
            # int8 codes + scales cross the reverse all-to-all (half the bytes of bf16)
            oq, osc = ulysses.ulysses_sla_attention_q8(q, k, v, L_global, attn_q8, group, TOKEN_ALIGN)
        else:
            o = ulysses.ulysses_sla_attention(q, k, v, L_global, attn, group, TOKEN_ALIGN)
            oq, osc = ops.quantize_blockwise(o.reshape(Lp, dim).contiguous(), 128, check_finite=False)
    else:
        # qkv lands head-major [3H, L, hd] straight from the GEMM epilogue (no permute);
        # the out-projection quantizes the head-major attention output in place
        qkv = ops.w8a8_gemm_ex(aq, asc, w.qkv.bt, w.qkv.scales, 128, None, torch.bfloat16, plane=hd)
        if hd == 128 and Lp >= 128:
            # the attention epilogue emits the out-projection's block-quantized
            # A operand (codes [L, H*hd] + scales) directly
            oq, osc = ops.sla_attention(qkv[:heads], qkv[heads:2 * heads], qkv[2 * heads:], sla["q_block"],
                                        sla["kv_block"], sla["topk_ratio"], sla.get("linear_mix", 1.0), True,
                                        out_dtype=torch.int8, pv_fp8=sla.get("pv_fp8", False))
        else:
            o = attn(qkv[:heads], qkv[heads:2 * heads], qkv[2 * heads:])           # [H, L, hd]
            oq, osc = ops.quantize_blockwise_planar(o)
    po = ops.w8a8_gemm(oq, osc, w.out_proj.bt, w.out_proj.scales, 128, None, torch.float32, exact=False)
    # x2 = x1 + po and the block-quantized LayerNorm(x2) (mlp_in's A operand);
    # x2 overwrites x1
    if fused_nq:
        x2, bq, bsc = ops.add_norm_quant(x1, po, None, 0.0, w.ln_gain, w.ln_offset, layer_norm=True, sum_out=x1)
    else:
        x2, b = ops.add_norm(x1, po, None, 0.0, w.ln_gain, w.ln_offset, layer_norm=True, sum_out=x1)
        bq, bsc = ops.quantize_blockwise(b, 128, check_finite=False)
    # mlp_in -> GELU -> block quantization for mlp_out, all in the GEMM epilogue
    hq, hsc = ops.w8a8_gemm_quant(bq, bsc, w.mlp_in.bt, w.mlp_in.scales, 128, None, act=1)
    p2 = ops.w8a8_gemm(hq, hsc, w.mlp_out.bt, w.mlp_out.scales, 128, None, torch.float32, exact=False)
    return x2, p2


def model_forward(x, sigma, layers, heads, sla, L_global, group=None):
    pending = None
    for w in layers:
        x, pending = block_forward(x, sigma, w, heads, sla, L_global, group, pending)
    return x + pending


def rcm_sample(layers, heads: int, sla: dict, x_init: torch.Tensor, noises: list, sigmas, group=None,
               L_global: int | None = None):
    """sampler.py:281-302 over device tensors: x = sigma0*eps0; x0 = f(x, s_i);
    x = x0 + s_{i+1}*eps_{i+1}; exactly len(sigmas)-1 model calls."""
    L_global = x_init.shape[0] if L_global is None else L_global
    x = float(sigmas[0]) * x_init
    x0 = x
    for i in range(len(sigmas) - 1):
        x0 = model_forward(x, float(sigmas[i]), layers, heads, sla, L_global, group)
        if sigmas[i + 1] > 0:
            x = x0 + float(sigmas[i + 1]) * noises[i]
    return x0

"""Attention time on DiT-derived q/k/v vs random inputs (diagnostic)."""
import os, sys, time, torch
sys.path.insert(0, os.getcwd())
from paper_2512_16093_b200 import dit, ops
L, DIM, H, FFN = 75600, 5120, 40, 13824
w = dit.random_layers(DIM, FFN, 1, seed=0)[0]
g = torch.Generator(device="cuda").manual_seed(1)
x = torch.randn((L, DIM), generator=g, device="cuda")
a = ops.rmsnorm(x + 0.5 * w.sigma_emb, w.rms_gain)
aq = ops.quantize_blockwise(a, 128, check_finite=False)
qkv = ops.w8a8_gemm(aq[0], aq[1], w.qkv.bt, w.qkv.scales, 128, None, torch.bfloat16, False)
qh, kh, vh = [t.view(L, H, 128).permute(1, 0, 2).contiguous() for t in qkv.split(DIM, dim=1)]
del x, a, aq, qkv
rq, rk, rv = (torch.randn((H, L, 128), generator=g, device="cuda").to(torch.bfloat16) for _ in range(3))
def one(q, k, v):
    torch.cuda.synchronize()
    s0 = torch.cuda.memory_stats()
    c0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ops.sla_attention(q, k, v, 128, 64, 0.1, 1.0, True, out_dtype=torch.bfloat16)
    e1.record()
    c1 = time.perf_counter()
    torch.cuda.synchronize()
    s1 = torch.cuda.memory_stats()
    return e0.elapsed_time(e1), (c1 - c0) * 1e3, s1["num_alloc_retries"] - s0["num_alloc_retries"], s1.get("num_device_alloc", 0) - s0.get("num_device_alloc", 0)
for name, args in (("dit", (qh, kh, vh)), ("randn", (rq, rk, rv)), ("dit", (qh, kh, vh)), ("randn", (rq, rk, rv))):
    for _ in range(3):
        print(name, "gpu ms %.2f  cpu ms %.2f  retries %d  device_allocs %d" % one(*args))
print(torch.cuda.memory_summary(abbreviated=True)[:1500])

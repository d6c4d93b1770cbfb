"""Benchmark of the TurboDiffusion hot path on B200 (contract: one JSON line on rank 0).

Default workload (N=1): SLA + Sage attention at the Wan2.1-14B-720P shape
(BASELINE.json configs[3]: 40 heads, 75600 tokens, d=128, top-k 10% ->
119/1182 kv blocks, q_block 128 / kv_block 64) -- one step = one full
``sla_attention`` call (pool/quant Q, k_mean, pool/quant K, top-k, V^T,
linear branch, fused tcgen05 sparse attention + combine) on inputs resident
in HBM.  metric = executed sparse-softmax work (attention_flop_report,
attention.py:441-448) / step time, in TOPS.  Inputs (3 x 774 MB bf16) exceed
the 126 MB L2, so no flush is needed between steps.

Secondary line items in the same JSON: the W8A8 GEMM sweep at the
Wan2.1-1.3B shapes (configs[1]) and the fused-kernel roofline.

N>1 (torchrun): Ulysses -- each rank holds a token shard [L/P, H, d] of
q/k/v, all-to-all to a head shard, attention on H/P heads, all-to-all back
(strong scaling: the global problem is fixed).

--impl reference: the CPU oracle port (oracle/oracle.py, numpy + the C
restatement) on the host cores, one head of the same workload per step.

Roofline denominators: the tensor-core peaks MEASURED on this pool's B200s by
tools/mma_peak.py (profiles/int8_fp8_peak.json: tcgen05 MMA-only INT8 / FP8 /
BF16, burst and sustained), HBM from MEASURED_PEAKS.json.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

H_, L_, D_ = 40, 75600, 128
QB, KVB, RATIO = 128, 64, 0.1
METRIC = "SLA-Sage attn TOPS & W8A8 GEMM TOPS at Wan2.1-14B-720P shapes, 1/2/4/8 B200"
# kernels one sla_attention step launches (bf16 tensor-core path with the linear branch):
# kv_part + raw K pooling (third stream), k_mean + K codes (side stream), Q pool/quant,
# top-k (+ coverage matrix), coverage GEMM, fused attention
# (profiles/r02_launches_sla_step.csv lists them per step)
LAUNCHES_PER_STEP = 7
UNIT = "TOPS"


def sparse_ops(H=H_, L=L_, d=D_, qb=QB, kvb=KVB, ratio=RATIO) -> int:
    """attention.py:441-448 sparse_softmax_flops (QK^T + PV over selected blocks)."""
    nkv = -(-L // kvb)
    count = math.ceil(ratio * nkv)
    return 4 * H * L * min(count * kvb, L) * d


def _find_num(d, *words, avoid=()):
    """First numeric value in a (nested) dict whose key path contains all `words`."""
    stack = [("", d)]
    while stack:
        path, x = stack.pop(0)
        if isinstance(x, dict):
            stack += [(f"{path}.{k}".lower(), v) for k, v in x.items()]
        elif isinstance(x, (int, float)) and all(w in path for w in words) and not any(a in path for a in avoid):
            return float(x)
    return None


def peaks():
    """(HBM GB/s, bf16 TFLOP/s burst, source).  MEASURED_PEAKS.json is driver-written per
    pod (key names are matched loosely); without it, the pool's measured figures that
    BASELINE.md section 3 copies from it (6547.2 GB/s, 1672.5 TFLOP/s burst)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        hbm = _find_num(p, "hbm") or _find_num(p, "gb")
        bf = (_find_num(p, "bf16", "burst") or _find_num(p, "bf16", avoid=("sustained",))
              or _find_num(p, "tflop", avoid=("sustained",)))
        if hbm and bf:
            return hbm, bf, "measured (MEASURED_PEAKS.json)"
    except Exception:
        pass
    return 6547.2, 1672.5, "measured (MEASURED_PEAKS.json values quoted in BASELINE.md)"


PEAK_FILE = os.path.join(ROOT, "profiles", "int8_fp8_peak.json")


def tc_peaks():
    """Measured tcgen05 MMA-only peaks (tools/mma_peak.py on this pool's B200s)
    -> {"int8": (burst, sustained), "fp8": ..., "bf16": ...} in TOPS, or None."""
    try:
        with open(PEAK_FILE) as f:
            s = json.load(f)["summary"]
        return {k: (s[f"{k}_tops_burst"], s[f"{k}_tops_sustained"]) for k in ("int8", "fp8", "bf16")}
    except Exception:
        return None


def mixed_peak(a: float, b: float) -> float:
    """Peak of work split evenly between two MMA kinds (QK^T and PV carry the
    same op count): time = ops/2/a + ops/2/b."""
    return 1.0 / (0.5 / a + 0.5 / b)


_REJECT_REASONS = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown")


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region: NVML polled
    every 10 ms from a thread (the timed region is ~100 ms, too short for
    `nvidia-smi -lms`), falling back to nvidia-smi when NVML is unavailable."""

    _REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
                ("sw_power_cap", 0x4), ("hw_power_brake_slowdown", 0x80))

    def __init__(self, index=0):
        self.index, self.rows, self.proc, self.nvml = index, [], None, None
        self.stop = threading.Event()

    def _poll(self):
        import pynvml as N
        h = N.nvmlDeviceGetHandleByIndex(self.index)
        mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
        while True:
            try:
                sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                rs = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                pw = N.nvmlDeviceGetPowerUsage(h) / 1e3
            except Exception:
                break
            row = [str(sm), str(mx), f"{pw:.1f}"]
            row += ["Active" if rs & bit else "Not Active" for name, bit in self._REASONS[:4]]
            self.rows.append(row)
            if self.stop.wait(0.01):
                break

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            self.nvml = True
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            time.sleep(0.05)
            return self
        except Exception:
            self.nvml = None
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.nvml:
            self.stop.set()
            self.t.join(timeout=2)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = [float(r[0]) for r in self.rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 7 and r[1].replace(".", "").isdigit()]
        reasons = set()
        for r in self.rows:
            if len(r) >= 7:
                for name, val in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                                      "sw_power_cap"), r[3:7]):
                    if val.lower() == "active":
                        reasons.add(name)
        pw = [float(r[2]) for r in self.rows if len(r) >= 7 and r[2].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w": statistics.median(pw) if pw else None,
                "source": "nvml" if self.nvml else "nvidia-smi"}


# --------------------------------------------------------------- reference arm

def _dropin_chunk():
    from paper_2512_16093_b200 import attention
    return attention._HOST_CHUNK_HEADS


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
    import numpy as np

    import gen
    from oracle import oracle as O
    cores = os.cpu_count() or 1
    q, k, v = gen.gaussian_qkv(2, 1, L_, D_, bf16=True)
    ops_head = sparse_ops(H=1)
    for _ in range(args.warmup if args.warmup <= 1 else 1):
        O.sla_attention(q[:, :8192], k[:, :8192], v[:, :8192], QB, KVB, RATIO, 1.0)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        O.sla_attention(q, k, v, QB, KVB, RATIO, 1.0)
        times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    val = ops_head / t / 1e12
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "cfg4 SLA attention, 1 of 40 heads per step (CPU oracle port)",
                       "heads": 1, "seq_len": L_, "head_dim": D_, "q_block": QB, "kv_block": KVB,
                       "topk_ratio": RATIO},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": "1 head x 75600 tokens of cfg4 per step (numpy/OpenBLAS oracle)"},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- our arm

def cpu_info():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    return model, os.cpu_count() or 1


def cpu_oracle_time(fn, threads=None):
    """Wall time of fn() on the host (BLAS threads limited when `threads`)."""
    from threadpoolctl import threadpool_limits
    if threads is None:
        t0 = time.perf_counter()
        r = fn()
        return time.perf_counter() - t0, r
    with threadpool_limits(threads):
        t0 = time.perf_counter()
        r = fn()
        return time.perf_counter() - t0, r


def parity(got, want):
    """cos / rel-L2 / rel-L1 of the GPU output against the oracle (f64)."""
    from oracle import oracle as O
    import numpy as np
    cos, rel2, rel1 = O.error_metrics(np.asarray(got, np.float32), np.asarray(want, np.float32))
    return {"cos": cos, "rel_l2": rel2, "rel_l1": rel1, "ok": bool(cos >= 0.999 and rel1 <= 1e-2)}


def cpu_baseline_cfg4(q0, k0, v0, gpu_out0):
    """Oracle port on head 0 of the bench's OWN cfg4 inputs (bf16 values, f32
    upcast), all host threads and one thread, plus the parity of the GPU
    output of that head from the timed step (~10-20 s, rank 0 only)."""
    from oracle import oracle as O
    model, cores = cpu_info()
    t_all, want = cpu_oracle_time(lambda: O.sla_attention(q0, k0, v0, QB, KVB, RATIO, 1.0))
    t_one, _ = cpu_oracle_time(lambda: O.sla_attention(q0, k0, v0, QB, KVB, RATIO, 1.0), threads=1)
    return {"value": sparse_ops(H=1) / t_all / 1e12, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"head 0 of this run's cfg4 inputs (1 of 40 heads, 75600 tokens), {t_all:.1f} s on "
                      f"{cores} threads, numpy/OpenBLAS oracle port; per-head work, so x40 heads = the step",
            "cpu_model": model, "value_1thread": sparse_ops(H=1) / t_one / 1e12, "seconds": t_all,
            "seconds_1thread": t_one, "parity_gpu_vs_oracle_head0": parity(gpu_out0, want)}


DIT_DIM, DIT_FFN, DIT_STEPS = 5120, 13824, 4


def dit_ops_per_layer(L=L_, dim=DIT_DIM, ffn=DIT_FFN, heads=H_):
    """Per layer per step: W8A8 projections 2*L*(dim*3dim + dim*dim + 2*dim*ffn)
    plus the SLA attention's executed work (attention_flop_report)."""
    return 2 * L * (dim * 3 * dim + dim * dim + 2 * dim * ffn) + sparse_ops(H=heads, L=L)


def bench_dit(world, rank, num_layers, pv_fp8=False, samples=3, tcp=None):
    """cfg5 latency: full rCM samples (4 steps x num_layers layers), seq-parallel
    linears + Ulysses attention across ranks; max over ranks of CUDA-event time,
    median of `samples` samples.  The initial state and the per-step noise are
    drawn for the WHOLE sequence from one seeded stream and each rank takes its
    token shard, so every N computes the same sample."""
    import torch
    import torch.distributed as dist
    from paper_2512_16093_b200 import dit, ulysses
    torch.cuda.empty_cache()
    layers = dit.random_layers(DIT_DIM, DIT_FFN, num_layers, seed=0)
    lo, hi = ulysses.token_bounds(L_, world, rank, dit.TOKEN_ALIGN)
    g = torch.Generator(device="cuda").manual_seed(77)

    def shard_of_global():
        full = torch.randn((L_, DIT_DIM), generator=g, device="cuda")
        part = full[lo:hi].clone()
        del full
        return part
    x_init = shard_of_global()
    noises = [shard_of_global() for _ in range(DIT_STEPS - 1)]
    sig = [80.0 * (0.5 / 80.0) ** (i / (DIT_STEPS - 1)) for i in range(DIT_STEPS)] + [0.0]   # make_schedule(4)
    sla = dict(q_block=QB, kv_block=KVB, topk_ratio=RATIO, linear_mix=1.0, pv_fp8=pv_fp8)
    if world > 1 and os.environ.get("TB_ULYSSES_P2P") == "1":
        ulysses.prepare_p2p(L_, H_, D_, None, dit.TOKEN_ALIGN)      # collective allocation at setup
    dit.block_forward(x_init, sig[0], layers[0], H_, sla, L_)          # warm-up (one block)
    torch.cuda.synchronize()
    lat = []
    out = None
    for _ in range(samples):
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = dit.rcm_sample(layers, H_, sla, x_init, noises, sig, L_global=L_)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if world > 1:
            t_ = torch.tensor([ms], device="cuda")
            dist.all_reduce(t_, op=dist.ReduceOp.MAX)
            ms = float(t_.item())
        lat.append(ms / 1e3)
    ops_total = dit_ops_per_layer() * num_layers * DIT_STEPS
    finite = bool(torch.isfinite(out).all().item())
    checksum = float(out.double().abs().sum().item())
    if world > 1:
        t_ = torch.tensor([checksum], device="cuda", dtype=torch.float64)
        dist.all_reduce(t_)
        checksum = float(t_.item())
    del layers, noises, out
    torch.cuda.empty_cache()
    med = statistics.median(lat)
    res = {"workload": "cfg5: rCM 4-step sample, Wan2.1-14B-720P-shaped toy DiT (dim 5120, 40 heads, "
                       f"FFN 13824, {num_layers} layers, L 75600), SLA 0.1 + Sage INT8 + W8A8",
           "latency_s": med, "latency_samples_s": lat, "ops": ops_total, "TOPS": ops_total / med / 1e12,
           "weights": "random-init on device (N(0,1)/sqrt(fan_in), block-quantized)", "finite": finite,
           "sample_abs_sum": checksum,
           "noise": "global [L, dim] state and noise from one seeded device stream, sliced per rank"}
    if tcp:
        lin = 2 * L_ * (DIT_DIM * 3 * DIT_DIM + DIT_DIM * DIT_DIM + 2 * DIT_DIM * DIT_FFN) * num_layers * DIT_STEPS
        att = ops_total - lin
        # bound: linears at the sustained INT8 peak, attention at the sustained INT8/BF16 mix
        t_bound = lin / (tcp["int8"][1] * 1e12) + att / (mixed_peak(tcp["int8"][1], tcp["bf16"][1]) * 1e12)
        res["roofline"] = {"bound_s": t_bound, "frac": t_bound / med / world,
                           "note": "per GPU: W8A8 work at the measured sustained INT8 MMA peak + attention "
                                   "work at the sustained INT8/BF16 mix (profiles/int8_fp8_peak.json)"}
    return res


def time_graph(fn, reps=10):
    """CUDA-graph the call, replay `reps` times; ms per replay (CUDA events)."""
    import torch
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    cap = torch.cuda.Stream()
    cap.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(cap):
        fn()
    torch.cuda.current_stream().wait_stream(cap)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        out = fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, out, g


def bench_configs(tcp, cpu: bool):
    """configs[0] (cfg1) and configs[2] (cfg3) at the reference default block
    sizes (64/64) and at q_block 128, and configs[3] (cfg4) at 64/64 (its
    q_block 128 form is the headline): device step time, executed-work TOPS,
    and (rank 0) the oracle on one head of the same inputs with parity."""
    import numpy as np
    import torch
    from paper_2512_16093_b200 import ops
    from oracle import oracle as O
    res = {}
    peak = mixed_peak(tcp["int8"][0], tcp["bf16"][0]) if tcp else None
    for (name, H, L, seed, qbs) in (("cfg1", 2, 4096, 11, (64, 128)), ("cfg3", 12, 32760, 12, (64, 128)),
                                    ("cfg4", 40, 75600, 13, (64,))):
        g = torch.Generator(device="cuda").manual_seed(seed)
        qkv = [torch.randn((H, L, D_), generator=g, device="cuda").to(torch.bfloat16) for _ in range(3)]
        for qb in qbs:
            ms, out, gr = time_graph(lambda: ops.sla_attention(qkv[0], qkv[1], qkv[2], qb, 64, RATIO, 1.0,
                                                               out_dtype=torch.bfloat16))
            ops_ = sparse_ops(H=H, L=L, qb=qb)
            r = {"heads": H, "seq_len": L, "q_block": qb, "kv_block": 64, "topk_ratio": RATIO,
                 "ms": ms, "TOPS": ops_ / (ms * 1e-3) / 1e12}
            if peak:
                r["frac_step_of_mixed_peak"] = r["TOPS"] / peak
            if cpu:
                h0 = [t[0:1].float().cpu().numpy() for t in qkv]
                tcpu, want = cpu_oracle_time(lambda: O.sla_attention(h0[0], h0[1], h0[2], qb, 64, RATIO, 1.0))
                r["cpu_baseline"] = {"value": sparse_ops(H=1, L=L, qb=qb) / tcpu / 1e12, "unit": UNIT,
                                     "seconds_per_head": tcpu, "sample": "head 0 of the same inputs",
                                     "kind": "port", "cores": os.cpu_count() or 1}
                r["parity_head0"] = parity(out[0:1].float().cpu().numpy(), want)
            del gr, out
            res[f"{name}_q{qb}"] = r
        del qkv
    return res


def bench_w8a8(tcp, hbm, cpu: bool):
    """configs[1]: the W8A8 sweep at M = 32760 (exact and fast promotion), the
    activation-quantization pass at those shapes, and the CPU
    quantized_linear_forward (oracle, the reference's sgemm-per-k-block order)
    on a 2048-row sample per shape."""
    import numpy as np
    import torch
    from paper_2512_16093_b200 import ops
    from oracle import oracle as O
    w8 = {}
    M = 32760
    i8 = tcp["int8"][0] if tcp else None
    for (K, N) in ((1536, 1536), (1536, 4608), (1536, 8960), (8960, 1536)):
        xq = torch.randint(-127, 128, (M, K), dtype=torch.int8, device="cuda")
        xs = torch.rand((-(-M // 128), K // 128), device="cuda") * 0.01
        bt = torch.randint(-127, 128, (N, K), dtype=torch.int8, device="cuda")
        bs = torch.rand((K // 128, N // 128), device="cuda") * 0.01
        res = {}
        for mode in ("exact", "fast"):
            fn = lambda: ops.w8a8_gemm(xq, xs, bt, bs, 128, exact=(mode == "exact"))
            for _ in range(3):
                fn()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                fn()
            e1.record()
            torch.cuda.synchronize()
            gms = e0.elapsed_time(e1) / 10
            tops = 2 * M * K * N / (gms * 1e-3) / 1e12
            res[mode] = {"ms": gms, "TOPS": tops, "frac_int8_peak": (tops / i8) if i8 else None}
        # full quantized_linear_forward: activation quant (bf16 x) + GEMM
        x = torch.randn((M, K), device="cuda").to(torch.bfloat16)
        fq = lambda: ops.quantize_blockwise(x, 128, check_finite=False)
        for _ in range(3):
            fq()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            fq()
        e1.record()
        torch.cuda.synchronize()
        qms = e0.elapsed_time(e1) / 10
        res["act_quant"] = {"ms": qms, "GBps": 3 * M * K / (qms * 1e-3) / 1e9,
                            "frac_hbm": 3 * M * K / (qms * 1e-3) / 1e9 / hbm,
                            "bytes": "2 B bf16 read + 1 B int8 written per element"}
        fl = lambda: ops.quantized_linear(x, bt, bs, 128, None, torch.float32, exact=True)
        for _ in range(3):
            fl()
        e0.record()
        for _ in range(10):
            fl()
        e1.record()
        torch.cuda.synchronize()
        lms = e0.elapsed_time(e1) / 10
        res["quantized_linear_forward"] = {"ms": lms, "TOPS": 2 * M * K * N / (lms * 1e-3) / 1e12}
        if cpu:
            rows = 2048
            xc = x[:rows].float().cpu().numpy()
            wq = bt.t().contiguous().cpu().numpy()
            ws = bs.cpu().numpy()

            def cpu_ql():
                aq, as_ = O.quantize_blockwise(xc, 128)
                return O.w8a8_blas(aq, as_, wq, ws, 128)
            tcpu, want = cpu_oracle_time(cpu_ql)
            got = ops.quantized_linear(x[:rows], bt, bs, 128, None, torch.float32, exact=True).cpu().numpy()
            res["cpu_baseline"] = {"value": 2 * rows * K * N / tcpu / 1e12, "unit": UNIT, "seconds": tcpu,
                                   "sample": f"{rows} of {M} rows (quantize_blockwise + w8a8 in the reference's "
                                             "numpy sgemm-per-k-block order)", "kind": "port",
                                   "cores": os.cpu_count() or 1,
                                   "bit_exact_gpu_vs_oracle": bool(np.array_equal(got, want))}
        w8[f"{K}x{N}"] = res
        del xq, xs, bt, bs, x
    w8["peak_note"] = ("fractions of the measured tcgen05 kind::i8 MMA-only burst peak "
                       f"{i8:.0f} TOPS (profiles/int8_fp8_peak.json)" if i8 else "no measured INT8 peak")
    return w8


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-w8a8", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the cfg1 / cfg3 lines")
    ap.add_argument("--heads", type=int, default=H_)
    ap.add_argument("--no-dit", action="store_true")
    ap.add_argument("--dit-samples", type=int, default=3)
    ap.add_argument("--no-fp8", action="store_true", help="skip the opt-in FP8 P/V measurement")
    ap.add_argument("--no-graph", action="store_true", help="eager launches in the timed region")
    ap.add_argument("--dit-layers", type=int, default=40)
    ap.add_argument("--dit-pv-fp8", action="store_true", help="DiT attention with the opt-in FP8 P/V (not the default)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("TB_BENCH_GLOO_CHECK") == "1":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1 and os.environ.get("TB_BENCH_GLOO_CHECK") == "1":
        # FUNCTIONAL CHECK ONLY (never a measurement): exercises the N>1 code path
        # (token shards, Ulysses exchanges, max-over-ranks) on a one-GPU box --
        # NCCL refuses two ranks on one device, so gloo with the exchange
        # staged through host memory (tests/test_gpu_dit_ulysses.py's shim)
        dist.init_process_group("gloo")
        _a2a = dist.all_to_all_single

        class _Done:
            def wait(self):
                return True

        def _staged(out, inp, group=None, async_op=False, **kw):
            h = torch.empty(out.shape, dtype=out.dtype)
            _a2a(h, inp.cpu(), group=group)
            out.copy_(h)
            return _Done() if async_op else None
        dist.all_to_all_single = _staged
    elif world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")         # communicator setup visible in the log (N ranks)
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2512_16093_b200 import _lib, ops, ulysses
    from paper_2512_16093_b200.attention import attention_flop_report, SLAConfig
    _lib.load(require_device=True)
    sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

    H = args.heads
    total_ops = sparse_ops(H=H)
    assert total_ops == attention_flop_report(L_, D_, H, SLAConfig(QB, KVB, RATIO)).sparse_softmax_flops
    # the global cfg4 problem from one seeded stream; each rank keeps its token
    # shard [L_p, H, d] of q/k/v (bf16), resident in HBM -- every N sees the same inputs
    lo, hi = ulysses.token_bounds(L_, world, rank)
    g = torch.Generator(device="cuda").manual_seed(1234)
    shard = []
    for _ in range(3):
        full = torch.randn((L_, H, D_), generator=g, device="cuda", dtype=torch.float32).to(torch.bfloat16)
        shard.append(full[lo:hi].clone())
        del full
    torch.cuda.empty_cache()

    def attn(qh, kh, vh):
        return ops.sla_attention(qh, kh, vh, QB, KVB, RATIO, 1.0, out_dtype=torch.bfloat16)

    def step():
        if world == 1:
            return attn(*head_major)                               # head-major copies resident in HBM
        return ulysses.ulysses_sla_attention(shard[0], shard[1], shard[2], L_, attn)

    head_major = [t.permute(1, 0, 2).contiguous() for t in shard] if world == 1 else None

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # N=1: the step (its ~10 launches over three streams) is captured once in a
    # CUDA graph and replayed, so host-side launch jitter cannot starve the GPU
    # inside the timed region; the e2e figure below stays an eager call.
    graph = None
    step_out = None
    if world == 1 and not args.no_graph:
        cap = torch.cuda.Stream()
        cap.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cap):
            step()
        torch.cuda.current_stream().wait_stream(cap)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step_out = step()
        for _ in range(2):
            graph.replay()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    remeasured = None
    for attempt in range(2):
        with ClockSampler(local) as clk:
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            ev0.record()
            for _ in range(args.steps):
                if graph is not None:
                    graph.replay()
                else:
                    step_out = step()
            ev1.record()
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
        # a timed region that saw a hardware / thermal slowdown is measured once more
        # (sw_power_cap is kept and noted); every rank takes the same decision
        bad = [r for r in clk.summary()["reasons"] if r in _REJECT_REASONS]
        flag = torch.tensor([1.0 if bad else 0.0], device="cuda")
        if world > 1:
            dist.all_reduce(flag, op=dist.ReduceOp.MAX)
        if attempt == 0 and flag.item() > 0:
            remeasured = bad or ["on another rank"]
            continue
        break
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = total_ops / (ms * 1e-3) / 1e12
    # head 0 of the timed step's output (parity against the oracle below)
    out_head0 = None
    if world == 1 and step_out is not None:
        out_head0 = step_out[0:1].float().cpu().numpy()
    elif world > 1 and step_out is not None:
        out_head0 = None

    # ---- dominant kernel (fused tcgen05 attention) timed alone on its stream
    hbm, bf16_peak, peak_kind = peaks()
    tcp = tc_peaks()
    if tcp:
        mixed = mixed_peak(tcp["int8"][0], tcp["bf16"][0])
        peak_note = (f"measured tcgen05 MMA-only burst peaks (profiles/int8_fp8_peak.json): INT8 QK^T at "
                     f"{tcp['int8'][0]:.0f} TOPS + BF16 PV at {tcp['bf16'][0]:.0f} TOPS, equal op counts")
    else:
        mixed = bf16_peak * 4.0 / 3.0
        peak_note = f"INT8 QK^T (2x) + BF16 PV at {peak_kind} cuBLAS bf16 burst {bf16_peak} TFLOP/s x 4/3"
    roof = None
    if world == 1:
        qh, kh, vh = head_major
        _, parts = ops.sla_attention(qh, kh, vh, QB, KVB, RATIO, 1.0, out_dtype=torch.bfloat16, return_parts=True)
        out = torch.empty((H, L_, D_), dtype=torch.bfloat16, device="cuda")
        a = ops.sla_args(q=ops.ptr(qh), k=ops.ptr(kh), v=ops.ptr(vh), dtype=1, H=H, L=L_, d=D_, q_block=QB,
                         kv_block=KVB, count=parts["count"], scale=1.0 / math.sqrt(D_), linear_mix=1.0, quantized=1,
                         q_codes=ops.ptr(parts["q_codes"]), k_codes=ops.ptr(parts["k_codes"]),
                         q_scales=ops.ptr(parts["q_scales"]), k_scales=ops.ptr(parts["k_scales"]),
                         k_mean=ops.ptr(parts["k_mean"]), idx=ops.ptr(parts["idx"]), vt=None,
                         l_pad=(-(-L_ // 64)) * 64, num_l=None, den_l=None, lin_ld=0, lin_hs=0,
                         lin_kv=ops.ptr(parts["lin_kv"]), lin_dx=parts["lin_kv"].shape[2],
                         out=ops.ptr(out), out_dtype=1, row_max=None, den=None)
        import ctypes
        lib = _lib.load()
        for _ in range(3):
            lib.tb_sla_attention(ctypes.byref(a), ops.stream_ptr())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        e0.record()
        for _ in range(reps):
            lib.tb_sla_attention(ctypes.byref(a), ops.stream_ptr())
        e1.record()
        torch.cuda.synchronize()
        kms = e0.elapsed_time(e1) / reps
        ach = total_ops / (kms * 1e-3) / 1e12
        traffic, tsrc = None, None
        for fn in ("r02_sla_tc_traffic.json", "r01_sla_tc_traffic.json"):
            try:        # dram read+write bytes per launch from the committed ncu --set full capture
                with open(os.path.join(ROOT, "profiles", fn)) as f:
                    traffic = json.load(f)["traffic_bytes"]
                tsrc = "profiles/" + fn
                break
            except Exception:
                pass
        roof = {"bound": "tensor", "achieved": ach, "peak": mixed, "unit": "TFLOP/s",
                "frac": ach / mixed, "traffic": traffic, "traffic_source": tsrc, "kernel": "sla_tc_kernel",
                "kernel_ms": kms, "share_of_step": kms / ms, "peak_note": peak_note}
        if tcp:
            roof["frac_of_int8_fp8_peak"] = ach / tcp["int8"][0]
            roof["frac_of_sustained_mix"] = ach / mixed_peak(tcp["int8"][1], tcp["bf16"][1])
        del out

    # ---- e2e through the drop-in (the call a turbobench user makes:
    # attention.sla_attention(AttnInputs(numpy f32 q, k, v), SLAConfig(...)) ->
    # numpy f32), host buffers in and out, every copy inside the timed region;
    # plus the torch API on pinned bf16 host tensors (ops.sla_attention_host)
    e2e = e2e_torch = None
    if world == 1:
        import numpy as np
        from paper_2512_16093_b200.attention import AttnInputs, sla_attention as dropin_sla
        hn = [t.float().cpu().numpy() for t in head_major]             # f32 numpy, as the reference takes
        cfg = SLAConfig(q_block=QB, kv_block=KVB, topk_ratio=RATIO, linear_mix=1.0)
        inp = AttnInputs(hn[0], hn[1], hn[2])
        for _ in range(2):              # the caching host allocator pins the result blocks once
            dropin_sla(inp, cfg)
        torch.cuda.synchronize()
        times = []
        for _ in range(3):
            t0 = time.perf_counter()
            o_np = dropin_sla(inp, cfg)                                # returns a host numpy array
            times.append(time.perf_counter() - t0)
        ems = statistics.median(times) * 1e3
        moved = dict(ops.LAST_HOST_TRANSFER)
        e2e = {"value": total_ops / (ems * 1e-3) / 1e12, "unit": UNIT, "ms_per_step": ems,
               "h2d_bytes_per_step": moved["h2d_bytes"], "d2h_bytes_per_step": o_np.nbytes,
               "api": "paper_2512_16093_b200.attention.sla_attention(AttnInputs(numpy f32), SLAConfig) -> numpy f32 "
                      "(drop-in for turbobench.attention.sla_attention); host wall clock, median of 3; per "
                      f"{_dropin_chunk()}-head chunk: numpy->pinned staging (next chunk on a worker thread), H2D, "
                      "attention, D2H straight into the page-locked result array",
               "h2d_bytes_note": (f"{moved['narrow_chunks']}/{moved['chunks']} head chunks had bf16-valued q and k "
                                  "(generator G: bf16-rounded Gaussians), detected on the fly while staging and "
                                  "uploaded as their exact bf16 bit patterns (lossless); V always crosses as bf16 "
                                  "(the kernels read V only as bf16)")}
        if out_head0 is not None:
            e2e["parity_vs_device_step_head0"] = parity(o_np[0:1], out_head0)
        # the same call on f32 q / k that are NOT bf16-valued (one ulp added to
        # every element): the f32 upload, 4 B per q / k element
        for x_ in (hn[0], hn[1]):
            x_.view(np.uint32)[...] |= 1
        dropin_sla(inp, cfg)
        times = []
        for _ in range(3):
            t0 = time.perf_counter()
            o_np = dropin_sla(inp, cfg)
            times.append(time.perf_counter() - t0)
        fms = statistics.median(times) * 1e3
        moved = dict(ops.LAST_HOST_TRANSFER)
        e2e["f32_valued_inputs"] = {"value": total_ops / (fms * 1e-3) / 1e12, "unit": UNIT, "ms_per_step": fms,
                                    "h2d_bytes_per_step": moved["h2d_bytes"], "d2h_bytes_per_step": o_np.nbytes,
                                    "narrow_chunks": moved["narrow_chunks"],
                                    "note": "q, k perturbed by one ulp (not bf16-exact): q, k f32 + v bf16 cross PCIe"}
        if out_head0 is not None:
            e2e["f32_valued_inputs"]["parity_vs_device_step_head0"] = parity(o_np[0:1], out_head0)
        del hn, inp, o_np
        hq = [t.cpu().pin_memory() for t in head_major]
        hout = torch.empty((H, L_, D_), dtype=torch.bfloat16).pin_memory()

        def e2e_step():
            # torch API on pinned bf16 host buffers: per-head-chunk H2D / attention / D2H pipeline
            ops.sla_attention_host(hq[0], hq[1], hq[2], QB, KVB, RATIO, 1.0, out=hout)
        e2e_step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n_e2e = max(2, min(args.steps, 5))
        e0.record()
        for _ in range(n_e2e):
            e2e_step()
        e1.record()
        torch.cuda.synchronize()
        tms = e0.elapsed_time(e1) / n_e2e
        e2e_torch = {"value": total_ops / (tms * 1e-3) / 1e12, "unit": UNIT, "ms_per_step": tms,
                     "h2d_bytes_per_step": sum(t.numel() * 2 for t in hq), "d2h_bytes_per_step": hout.numel() * 2,
                     "api": "ops.sla_attention_host on pinned bf16 host tensors (CUDA events)"}
        del hq, hout
    else:
        # N > 1: each rank's token shard of q/k/v from pinned host memory, the
        # Ulysses attention (exchange, head-shard attention, exchange back), and
        # the token-shard output back to pinned host memory; max over ranks.
        # Bytes are per rank (every rank moves its own shard).
        hq = [t.cpu().pin_memory() for t in shard]
        hout = torch.empty(shard[0].shape, dtype=torch.bfloat16).pin_memory()
        dq = [torch.empty_like(t) for t in shard]

        def e2e_step():
            for d_, h_ in zip(dq, hq):
                d_.copy_(h_, non_blocking=True)
            o = ulysses.ulysses_sla_attention(dq[0], dq[1], dq[2], L_, attn)
            hout.copy_(o, non_blocking=True)
        e2e_step()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n_e2e = max(2, min(args.steps, 5))
        e0.record()
        for _ in range(n_e2e):
            e2e_step()
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / n_e2e], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ems = float(t.item())
        e2e = {"value": total_ops / (ems * 1e-3) / 1e12, "unit": UNIT, "ms_per_step": ems,
               "h2d_bytes_per_step": sum(t_.numel() * 2 for t_ in hq), "d2h_bytes_per_step": hout.numel() * 2,
               "bytes_note": "per rank", "api": "ulysses_sla_attention from pinned bf16 token shards"}
        del hq, hout, dq

    # ---- W8A8 GEMM sweep (configs[1]) + act-quant + CPU quantized_linear_forward
    w8 = None
    if world == 1 and not args.no_w8a8:
        w8 = bench_w8a8(tcp, hbm, cpu=not args.no_cpu_baseline)

    # ---- configs[0] / configs[2] lines (cfg1, cfg3) at 64/64 and 128/64
    cfgs = None
    if world == 1 and not args.no_configs:
        cfgs = bench_configs(tcp, cpu=not args.no_cpu_baseline)

    # ---- cfg5: full rCM 4-step sampling of the Wan2.1-14B-720P-shaped toy DiT
    dit_res = None
    if not args.no_dit:
        del shard
        head_major_keep = head_major
        head_major = None
        dit_res = bench_dit(world, rank, args.dit_layers, args.dit_pv_fp8, args.dit_samples, tcp)
        head_major = head_major_keep
        if args.dit_pv_fp8:
            dit_res["workload"] += " (opt-in FP8 P/V)"

    # ---- opt-in FP8 P/V: the same step and the fused kernel
    # alone with e4m3 P and V (kind::f8f6f4 PV), after the DiT sample so the
    # headline measurements run exactly as without it.  Reported beside the BF16
    # headline, not as it: FP8 P/V misses rel-L1 <= 1e-2 when the sparse
    # branch dominates (tests/test_gpu_parity.py).
    fp8 = None
    if world == 1 and not args.no_fp8:
        qh, kh, vh = head_major
        f8ms, _, g8 = time_graph(lambda: ops.sla_attention(qh, kh, vh, QB, KVB, RATIO, 1.0,
                                                           out_dtype=torch.bfloat16, pv_fp8=True), args.steps)
        del g8
        v8, v8s = ops.quant_v_fp8(vh)
        a.v_fp8, a.v_scales = ops.ptr(v8), ops.ptr(v8s)
        out = torch.empty((H, L_, D_), dtype=torch.bfloat16, device="cuda")
        a.out = ops.ptr(out)
        for _ in range(3):
            lib.tb_sla_attention(ctypes.byref(a), ops.stream_ptr())
        e0.record()
        for _ in range(reps):
            lib.tb_sla_attention(ctypes.byref(a), ops.stream_ptr())
        e1.record()
        torch.cuda.synchronize()
        f8k = e0.elapsed_time(e1) / reps
        a.v_fp8 = a.v_scales = None
        f8peak = mixed_peak(tcp["int8"][0], tcp["fp8"][0]) if tcp else bf16_peak * 2.0
        fp8 = {"step_ms": f8ms, "TOPS": total_ops / (f8ms * 1e-3) / 1e12, "kernel_ms": f8k,
               "kernel_TOPS": total_ops / (f8k * 1e-3) / 1e12, "peak": f8peak,
               "frac": total_ops / (f8k * 1e-3) / 1e12 / f8peak,
               "note": "opt-in (pv_fp8=True); e4m3 P + per-head-scaled e4m3 V; rel-L1 ~2e-2 when sparse-dominated; "
                       "peak = measured INT8 QK^T + FP8 PV MMA-only burst mix"}
        del out, v8, v8s

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline and out_head0 is not None:
            h0 = [t[0:1].float().cpu().numpy() for t in head_major]
            cpu = cpu_baseline_cfg4(h0[0], h0[1], h0[2], out_head0)
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "int8/bf16", "data": "synthetic",
                "config": {"workload": "cfg4: SLA+Sage attention, Wan2.1-14B-720P shape (configs[3])",
                           "heads": H, "seq_len": L_, "head_dim": D_, "q_block": QB, "kv_block": KVB,
                           "topk_ratio": RATIO, "parallelism": f"ulysses{world}",
                           "l2": "inputs 3 x 774 MB bf16 > 126 MB L2 (no flush needed)",
                           "launch": "CUDA graph replay of the step" if graph is not None else "eager"},
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "e2e_torch_pinned": e2e_torch,
                "w8a8": w8, "configs": cfgs, "fp8_pv": fp8,
                "dit": dit_res, "tc_peaks": tcp, "gpu_launches": LAUNCHES_PER_STEP * args.steps,
                "clocks": dict(clk.summary(), **({"remeasured_after": remeasured} if remeasured else {}))}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""Measure this B200's dense tensor-core peaks (tcgen05, MMA-only) -> profiles/int8_fp8_peak.json.

    python tools/mma_peak.py [--out profiles/int8_fp8_peak.json] [--sustain-s 4]

For kind::i8, kind::f16 (bf16) and kind::f8f6f4 (e4m3), cta_group::1 (M128
N256) and cta_group::2 (M256 N256), all 148 SMs issue back-to-back MMAs from
shared memory (tools/mma_peak.cu).  burst = best of 5 single launches of
~25 ms (CUDA events); sustained = launches back to back for --sustain-s
seconds (the power-capped figure that applies to a kernel timed inside a long
step).  NVML SM clocks and throttle reasons are sampled during each phase.
bench.py reads the result for its roofline denominators.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libmma_peak.so")
KINDS = {0: ("int8", 32), 1: ("bf16", 16), 2: ("fp8_e4m3", 32)}


def build():
    src = os.path.join(HERE, "mma_peak.cu")
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(src):
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                               "-shared", "-Xcompiler", "-fPIC", "-o", LIB, src])


class Clocks:
    def __init__(self):
        import pynvml as N
        N.nvmlInit()
        self.N, self.h = N, N.nvmlDeviceGetHandleByIndex(0)
        self.rows, self.stop = [], threading.Event()

    def __enter__(self):
        self.rows = []
        self.stop.clear()
        self.t = threading.Thread(target=self._poll, daemon=True)
        self.t.start()
        return self

    def _poll(self):
        N = self.N
        while not self.stop.is_set():
            sm = N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM)
            rs = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            pw = N.nvmlDeviceGetPowerUsage(self.h) / 1e3
            self.rows.append((sm, rs, pw))
            self.stop.wait(0.01)

    def __exit__(self, *exc):
        self.stop.set()
        self.t.join()

    def summary(self):
        names = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown"}
        reasons = sorted({n for _, rs, _ in self.rows for bit, n in names.items() if rs & bit})
        return {"sm_mhz_median": statistics.median([r[0] for r in self.rows]) if self.rows else None,
                "power_w_median": statistics.median([r[2] for r in self.rows]) if self.rows else None,
                "reasons": reasons, "samples": len(self.rows)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "int8_fp8_peak.json"))
    ap.add_argument("--sustain-s", type=float, default=4.0)
    args = ap.parse_args()
    build()
    import torch
    lib = ctypes.CDLL(LIB)
    lib.tb_mma_peak_launch.argtypes = [ctypes.c_int] * 4 + [ctypes.c_void_p]
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    st = torch.cuda.current_stream()
    clk = Clocks()
    N_ = 256
    res = {"device": torch.cuda.get_device_name(0), "sms": sms,
           "sm_max_mhz": clk.N.nvmlDeviceGetMaxClockInfo(clk.h, clk.N.NVML_CLOCK_SM),
           "method": "tcgen05.mma back to back from shared memory on every SM (no loads, no epilogue), "
                     "N=256, K=32 bytes per instruction, two alternating TMEM accumulators; burst = best of 5 "
                     "launches (~25 ms each), sustained = launches back to back for %.0f s; CUDA events, NVML "
                     "clocks sampled during each phase (tools/mma_peak.py)" % args.sustain_s,
           "peaks": {}}

    def run(kind, cg, iters):
        rc = lib.tb_mma_peak_launch(kind, cg, sms - sms % cg, iters, ctypes.c_void_p(st.cuda_stream))
        if rc != 0:
            raise RuntimeError(f"launch failed: cudaError {rc}")

    for kind in (0, 2, 1):
        name, kdim = KINDS[kind]
        for cg in (1, 2):
            ctas = sms - sms % cg
            flop_per_iter = 2 * 128 * N_ * kdim * ctas          # per CTA 128 rows of M
            run(kind, cg, 64)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            run(kind, cg, 4096)
            e1.record()
            torch.cuda.synchronize()
            iters = max(8, int(4096 * 25.0 / e0.elapsed_time(e1)) // 8 * 8)     # ~25 ms launches
            best = None
            with clk:
                for _ in range(5):
                    e0.record()
                    run(kind, cg, iters)
                    e1.record()
                    torch.cuda.synchronize()
                    ms = e0.elapsed_time(e1)
                    best = ms if best is None else min(best, ms)
            burst_clk = clk.summary()
            time.sleep(1.0)                                      # let the power state settle between phases
            n = 0
            with clk:
                e0.record()
                t0 = time.perf_counter()
                while time.perf_counter() - t0 < args.sustain_s:
                    for _ in range(8):
                        run(kind, cg, iters)
                    n += 8
                    torch.cuda.synchronize()
                e1.record()
                torch.cuda.synchronize()
            sus_ms = e0.elapsed_time(e1) / n
            sus_clk = clk.summary()
            burst = flop_per_iter * iters / (best * 1e-3) / 1e12
            sus = flop_per_iter * iters / (sus_ms * 1e-3) / 1e12
            per_clk = flop_per_iter * iters / (best * 1e-3) / (burst_clk["sm_mhz_median"] * 1e6) / ctas
            key = f"{name}_cg{cg}"
            res["peaks"][key] = {"burst_tops": burst, "sustained_tops": sus, "burst_ms": best,
                                 "sustained_ms_per_launch": sus_ms, "launches_sustained": n,
                                 "ops_per_clk_per_sm_at_burst": per_clk,
                                 "clocks_burst": burst_clk, "clocks_sustained": sus_clk}
            print(key, json.dumps(res["peaks"][key]), flush=True)
            time.sleep(1.0)
    p = res["peaks"]
    res["summary"] = {
        "int8_tops_burst": max(p["int8_cg1"]["burst_tops"], p["int8_cg2"]["burst_tops"]),
        "int8_tops_sustained": max(p["int8_cg1"]["sustained_tops"], p["int8_cg2"]["sustained_tops"]),
        "fp8_tops_burst": max(p["fp8_e4m3_cg1"]["burst_tops"], p["fp8_e4m3_cg2"]["burst_tops"]),
        "fp8_tops_sustained": max(p["fp8_e4m3_cg1"]["sustained_tops"], p["fp8_e4m3_cg2"]["sustained_tops"]),
        "bf16_tops_burst": max(p["bf16_cg1"]["burst_tops"], p["bf16_cg2"]["burst_tops"]),
        "bf16_tops_sustained": max(p["bf16_cg1"]["sustained_tops"], p["bf16_cg2"]["sustained_tops"]),
    }
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res["summary"]))


if __name__ == "__main__":
    sys.exit(main())

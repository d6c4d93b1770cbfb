"""cfg4 step (CUDA graph replay), k_mean and kv_part (with the K pool) alone for library variants given as
TB200_LIB paths on the command line (interleaved, 3 rounds); tools only."""
import os
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] == "--child":
    import torch
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2512_16093_b200 import ops  # noqa: E402
    H, L, D = 40, 75600, 128
    g = torch.Generator(device="cuda").manual_seed(0)
    q, k, v = (torch.randn((H, L, D), generator=g, device="cuda").to(torch.bfloat16) for _ in range(3))

    def graph_ms(fn, reps=10):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            fn()
        for _ in range(3):
            gr.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            gr.replay()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    step = graph_ms(lambda: ops.sla_attention(q, k, v, 128, 64, 0.1, 1.0, out_dtype=torch.bfloat16))
    km = graph_ms(lambda: ops.kmean(k))
    kvp = graph_ms(lambda: ops.linear_kv_part(k, v, 64, pool=True))
    print(f"{step:.3f} {km:.3f} {kvp:.3f}")
    sys.exit(0)

libs = sys.argv[1:]
res = {l: [] for l in libs}
for _ in range(3):
    for lib in libs:
        env = dict(os.environ)
        if lib != "base":
            env["TB200_LIB"] = lib
        out = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True, text=True)
        line = [x for x in out.stdout.splitlines() if x.strip()]
        res[lib].append(line[-1] if line else out.stderr[-300:])
for lib, r in res.items():
    print(os.path.basename(lib), "step ms / k_mean ms / kv_part ms:", r)

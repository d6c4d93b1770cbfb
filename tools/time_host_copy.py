"""Host-side copy rates that bound the drop-in's numpy e2e path (tools only):
numpy -> pinned staging memcpy (torch copy_, per thread count), pinned and
pageable H2D / D2H."""
import time

import numpy as np
import torch

n = 155 * 1024 * 1024 // 4          # one 4-head cfg4 f32 chunk of one tensor
src = np.random.default_rng(0).standard_normal(n, dtype=np.float32)
pin = torch.empty(n, dtype=torch.float32, pin_memory=True)
dev = torch.empty(n, dtype=torch.float32, device="cuda")
print("torch threads", torch.get_num_threads())
for th in (1, 4, 8, 16, torch.get_num_threads()):
    torch.set_num_threads(th)
    t0 = time.perf_counter()
    for _ in range(5):
        pin.copy_(torch.from_numpy(src))
    dt = (time.perf_counter() - t0) / 5
    print(f"numpy->pinned copy_ threads {th}: {n * 4 / dt / 1e9:.1f} GB/s")
t0 = time.perf_counter()
for _ in range(5):
    np.copyto(pin.numpy(), src)
print(f"np.copyto: {n * 4 / ((time.perf_counter() - t0) / 5) / 1e9:.1f} GB/s")
for name, s in (("pinned", pin), ("pageable", torch.from_numpy(src))):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        dev.copy_(s, non_blocking=True)
    torch.cuda.synchronize()
    print(f"H2D {name}: {n * 4 * 5 / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
out = np.empty_like(src)
for name, d in (("pinned", pin), ("pageable", torch.from_numpy(out))):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        d.copy_(dev, non_blocking=True)
    torch.cuda.synchronize()
    print(f"D2H {name}: {n * 4 * 5 / (time.perf_counter() - t0) / 1e9:.1f} GB/s")

# page-locking the caller's buffer in place instead of staging through pinned memory
cudart = torch.cuda.cudart()
big = np.random.default_rng(1).standard_normal(4 * n, dtype=np.float32)
for rep in range(2):
    t0 = time.perf_counter()
    rc = cudart.cudaHostRegister(big.ctypes.data, big.nbytes, 0)
    t1 = time.perf_counter()
    d2 = torch.empty(4 * n, dtype=torch.float32, device="cuda")
    d2.copy_(torch.from_numpy(big), non_blocking=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    cudart.cudaHostUnregister(big.ctypes.data)
    t3 = time.perf_counter()
    print(f"cudaHostRegister {big.nbytes / 1e9:.2f} GB: rc {rc}, register {(t1 - t0) * 1e3:.1f} ms "
          f"({big.nbytes / (t1 - t0) / 1e9:.1f} GB/s), H2D {big.nbytes / (t2 - t1) / 1e9:.1f} GB/s, "
          f"unregister {(t3 - t2) * 1e3:.1f} ms")

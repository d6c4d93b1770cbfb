import sys
import numpy as np
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests/golden")
import gen
from oracle import oracle as O
from paper_2512_16093_b200 import ops
for (M, K, N) in ((256, 1536, 384), (300, 512, 256), (128, 256, 256)):
    x = gen.gaussian_matrix(5, M, K); w = gen.gaussian_matrix(6, K, N, 1.0 / np.sqrt(K))
    wq, ws = O.quantize_blockwise(w, 128); xq, xs = O.quantize_blockwise(x, 128)
    want = O.w8a8(xq, xs, wq, ws, 128)
    bt = ops.transpose_codes(torch.from_numpy(wq).cuda())
    got = ops.w8a8_gemm(torch.from_numpy(xq).cuda(), torch.from_numpy(xs).cuda(), bt, torch.from_numpy(ws).cuda(), 128).cpu().numpy()
    d = np.abs(got - want)
    ulp = np.spacing(np.abs(want).astype(np.float32))
    print(M, K, N, "mism", int((got != want).sum()), "max abs", float(d.max()), "max ulps", float((d / ulp).max()),
          "rel", float(d.max() / np.abs(want).max()))
    bad = np.argwhere(got != want)[:3]
    for r, c in bad: print("  ", r, c, got[r, c], want[r, c])

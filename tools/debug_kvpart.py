import sys, os
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16093_b200 import _lib, ops
_lib.load(require_device=True)
H, L, d = 1, 64, 128
def run(k, v):
    kb = torch.tensor(k, dtype=torch.float32).reshape(1, L, d).cuda().to(torch.bfloat16)
    vb = torch.tensor(v, dtype=torch.float32).reshape(1, L, d).cuda().to(torch.bfloat16)
    dx = ops.linear_kv_dx(d)
    out = torch.empty((1, 1, dx, d), dtype=torch.bfloat16, device="cuda")
    ops.call("tb_linear_kv_part", ops.ptr(kb), ops.ptr(vb), H, L, d, 64, dx, ops.ptr(out), ops.stream_ptr())
    torch.cuda.synchronize()
    return out.float().cpu().numpy()[0, 0]
t = np.arange(L)[:, None] * np.ones((1, d)); c = np.ones((L, 1)) * np.arange(d)[None, :]
o = run(np.zeros((L, d)) - 20, c)   # phi ~ 0 -> expect ~0
print("phi~0:", np.abs(o[:d]).max())
o = run(np.zeros((L, d)), c / 8)     # phi = 1: num[v][kc] = 64 * v/8 = 8v
print("V=c/8, phiK=1: row v=0..5, cols 0..5\n", o[:6, :6], "\nrows 64..66:", o[64:67, :4], "\nden row", o[d, :6])
o = run(np.zeros((L, d)), t / 8)     # num = sum_t t/8 = 252
print("V=t/8:", o[:3, :6])
kk = np.full((L, d), -30.0); kk[5, :] = 0.0   # phi(K) = one-hot at token 5 (phi(-30) ~ 0)
o = run(kk, c / 8)                   # num[v][kc] = V[5][v] = v/8
print("phiK onehot token5, V=c/8:", o[:6, :4], o[100, :4])
kk = np.full((L, d), -30.0); kk[:, 7] = 0.0   # phi(K)[t][7] = 1, else 0 -> num[v][7] = sum_t V[t][v], other cols 0
o = run(kk, c / 8)
print("phiK col7: nonzero cols of row 8:", np.nonzero(np.abs(o[8]) > 1e-3)[0], o[8, 7])
for tok in (0, 1, 5, 8, 9, 17, 33, 63):
    kk = np.full((L, d), -30.0); kk[tok, :] = 0.0
    o = run(kk, t)                   # expect num = tok everywhere
    print("onehot tok", tok, "-> got", o[0, 0], o[70, 3], o[127, 127])

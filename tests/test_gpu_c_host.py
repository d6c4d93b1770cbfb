"""The C ABI from a plain C host: tests/c/sla_forward_host.c (no Python, no
torch in the process) is compiled with gcc against include/tb_capi.h and
libtb200.so, runs tb_sla_workspace_bytes + tb_sla_forward on inputs written
here, and its output must equal ops.sla_attention on the same inputs bit for
bit (q_block 128 and the reference default 64)."""
import os
import subprocess

import numpy as np
import pytest
import torch

import gen

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2512_16093_b200")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


@pytest.fixture(scope="module")
def host_bin(tmp_path_factory):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = str(tmp_path_factory.mktemp("chost") / "sla_forward_host")
    subprocess.run(["gcc", "-O2", os.path.join(ROOT, "tests", "c", "sla_forward_host.c"), "-o", out,
                    "-I", os.path.join(ROOT, "include"), "-I", os.path.join(CUDA, "include"),
                    "-L", PKG, "-ltb200", "-L", os.path.join(CUDA, "lib64"), "-lcudart", "-lm",
                    f"-Wl,-rpath,{PKG}"], check=True)
    return out


@pytest.mark.parametrize("qb", [128, 64])
def test_c_host_sla_forward_matches_device_op(host_bin, tmp_path, qb):
    from paper_2512_16093_b200 import ops
    H, L = 2, 3000
    q, k, v = gen.gaussian_qkv(31, H, L, 128, bf16=True)
    files = []
    for name, a in (("q", q), ("k", k), ("v", v)):
        t = torch.from_numpy(a).to(torch.bfloat16)
        p = tmp_path / f"{name}.bin"
        p.write_bytes(t.view(torch.int16).numpy().tobytes())
        files.append(str(p))
    outp = str(tmp_path / "out.bin")
    r = subprocess.run([host_bin, str(H), str(L), str(qb), *files, outp], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    got = np.fromfile(outp, dtype=np.float32).reshape(H, L, 128)
    dq, dk, dv = (torch.from_numpy(a).cuda().to(torch.bfloat16) for a in (q, k, v))
    want = ops.sla_attention(dq, dk, dv, qb, 64, 0.1, 1.0, out_dtype=torch.float32).cpu().numpy()
    assert np.array_equal(got, want)

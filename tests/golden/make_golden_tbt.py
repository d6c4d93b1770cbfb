"""Generate TBT1 tensor-file / manifest fixtures with the UNMODIFIED reference
(run in the build container, where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_tbt.py

Writes tests/golden/tbt/{float,quantized}/ : a 1-layer toy model (dim 32) through
turbobench.tensor_store.write_manifest, and its `turbobench quantize` output
(cli.py:24-39), plus tests/golden/tbt/forward.npz = the reference model's
forward on a fixed input for both manifests."""
import os
import shutil

import numpy as np
from turbobench.cli import main
from turbobench.sampler import model_from_manifest, make_random_weights, model_to_tensors
from turbobench.tensor_store import load_manifest, write_manifest

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "tbt")
shutil.rmtree(OUT, ignore_errors=True)
os.makedirs(OUT)
layers = make_random_weights(32, num_layers=1, seed=5)
meta = {"heads": 4, "model_dim": 32, "num_layers": 1, "num_steps": 3}
write_manifest(os.path.join(OUT, "float"), model_to_tensors(layers), metadata=meta, name="toy")
assert main(["quantize", os.path.join(OUT, "float"), "--block", "128", "--out", os.path.join(OUT, "quantized")]) == 0
x = np.random.default_rng(0).standard_normal((8, 32)).astype(np.float32)
res = {"x": x}
for kind in ("float", "quantized"):
    m = load_manifest(os.path.join(OUT, kind))
    res[kind] = model_from_manifest(m)(x, 1.0)
np.savez(os.path.join(OUT, "forward.npz"), **res)
print(sorted(os.listdir(os.path.join(OUT, "quantized"))))

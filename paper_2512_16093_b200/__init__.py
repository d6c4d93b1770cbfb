"""B200-native (sm_100a) TurboDiffusion hot path, drop-in for turbobench's operator API.

Modules mirror the reference (/root/reference/pkg/src/turbobench):
``attention`` (SLA / Sage attention), ``blockquant`` (block INT8, W8A8),
``sampler`` (rCM consistency sampling over a toy DiT) and ``ulysses``
(head-parallel sharding).  All compute runs in ``libtb200.so``.
"""
from . import _lib  # noqa: F401

__version__ = "0.1.0"


def __getattr__(name):
    # lazy submodule import keeps `import paper_2512_16093_b200` cheap
    import importlib
    if name in ("attention", "blockquant", "sampler", "ops", "ulysses", "tensor_store", "merge"):
        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)

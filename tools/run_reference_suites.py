"""Run the reference's OWN test suites and invariant suite against the drop-in
 -- test infrastructure, not product.

Two steps, because the reference exists only in the build container and the
drop-in needs a B200:

    # here: stage the reference's pkg/tests and its verify/bench/cli modules into
    # oracle/_ref/suites/ (git-ignored like every oracle/_ref artefact; nothing
    # under it is committed)
    python tools/run_reference_suites.py stage

    # on the GPU box (gpurun): alias turbobench.{attention,blockquant,sampler,
    # merge,tensor_store} to the drop-in, load the
    # staged reference modules on top of them, run pytest on the staged tests
    python tools/run_reference_suites.py run [pytest args]

The summary (per-file pass/fail counts, failures with their reason) is written
to gpurun_out/reference_suites.log; the committed copy lives in profiles/.
"""
from __future__ import annotations

import importlib.util
import os
import shutil
import sys
import types

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
STAGE = os.path.join(ROOT, "oracle", "_ref", "suites")
REF = "/root/reference/pkg"
DROPIN = ("attention", "blockquant", "sampler", "merge", "tensor_store")
REF_ONLY = ("verify", "bench", "cli")          # reference harness modules, run over the aliased drop-in


def stage():
    if os.path.isdir(STAGE):
        shutil.rmtree(STAGE)
    os.makedirs(os.path.join(STAGE, "tests"))
    os.makedirs(os.path.join(STAGE, "modules"))
    for f in sorted(os.listdir(os.path.join(REF, "tests"))):
        if f.endswith(".py"):
            shutil.copy(os.path.join(REF, "tests", f), os.path.join(STAGE, "tests", f))
    for m in REF_ONLY:
        shutil.copy(os.path.join(REF, "src", "turbobench", m + ".py"), os.path.join(STAGE, "modules", m + ".py"))
    print("staged", sorted(os.listdir(os.path.join(STAGE, "tests"))), "+", REF_ONLY, "->", STAGE)


def install_alias():
    """turbobench -> the drop-in, exactly as INTEGRATION.md section 1 shows,
    plus the reference's own verify/bench/cli modules resolved against it."""
    sys.path.insert(0, ROOT)
    import paper_2512_16093_b200 as pkg
    from paper_2512_16093_b200 import attention, blockquant, merge, sampler, tensor_store  # noqa: F401
    tb = types.ModuleType("turbobench")
    tb.__path__ = []
    tb.__version__ = "0.1.0+b200"
    sys.modules["turbobench"] = tb
    for m in DROPIN:
        mod = getattr(pkg, m)
        sys.modules["turbobench." + m] = mod
        setattr(tb, m, mod)
    for m in REF_ONLY:
        spec = importlib.util.spec_from_file_location("turbobench." + m, os.path.join(STAGE, "modules", m + ".py"))
        mod = importlib.util.module_from_spec(spec)
        mod.__package__ = "turbobench"
        sys.modules["turbobench." + m] = mod
        spec.loader.exec_module(mod)
        setattr(tb, m, mod)
    tb.__all__ = list(DROPIN + REF_ONLY)


class _Summary:
    def __init__(self):
        self.by_file, self.failures = {}, []

    def pytest_runtest_logreport(self, report):
        if report.when != "call" and not (report.when == "setup" and report.outcome != "passed"):
            return
        f = report.nodeid.split("::")[0]
        d = self.by_file.setdefault(f, {"passed": 0, "failed": 0, "skipped": 0})
        d[report.outcome] = d.get(report.outcome, 0) + 1
        if report.outcome == "failed":
            msg = str(report.longrepr).strip().splitlines()
            self.failures.append((report.nodeid, msg[-1][:300] if msg else ""))


def run(extra):
    import pytest
    install_alias()
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    summ = _Summary()
    rc = pytest.main([os.path.join(STAGE, "tests"), "-q", "-p", "no:cacheprovider", "--rootdir", STAGE,
                      "-o", "python_files=test_*.py"] + extra, plugins=[summ])
    lines = ["reference suites (/root/reference/pkg/tests + verify.py) against paper_2512_16093_b200 "
             "(turbobench.* aliased to the drop-in)", f"pytest rc {int(rc)}"]
    tot = {"passed": 0, "failed": 0, "skipped": 0}
    for f, d in sorted(s for s in summ.by_file.items()):
        lines.append(f"{os.path.basename(f):24s} passed {d.get('passed', 0):3d}  failed {d.get('failed', 0):3d}  "
                     f"skipped {d.get('skipped', 0):3d}")
        for k in tot:
            tot[k] += d.get(k, 0)
    lines.append(f"{'TOTAL':24s} passed {tot['passed']:3d}  failed {tot['failed']:3d}  skipped {tot['skipped']:3d}")
    for nid, msg in summ.failures:
        lines.append(f"FAILED {nid}: {msg}")
    text = "\n".join(lines)
    with open(os.path.join(ROOT, "gpurun_out", "reference_suites.log"), "w") as f:
        f.write(text + "\n")
    print(text)
    return int(rc)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "stage":
        stage()
    else:
        sys.exit(run(sys.argv[2:]))

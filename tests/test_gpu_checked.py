"""The production and oracle-mode suites against a ZF_CHECKS=1 build of the
library (device-side traps on any queue slot outside the queue, round-scratch
index outside the warp's records, store outside the output, or a round that
reads the pack before its bulk copy landed).  compute-sanitizer is closed on
the GPU pool, so these checks are the race/bounds evidence for the shared
memory queue, the cooperative round scratch and the split staging."""
import os
import pathlib
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = pathlib.Path(__file__).resolve().parents[1]


def test_suites_pass_on_checked_build(cuda):
    lib = ROOT / "build" / "variants" / "checked.so"
    if not lib.exists():
        from paper_1403_6870_b200 import _build
        lib = _build.build_variant("checked", ["ZF_CHECKS=1"])
    env = dict(os.environ, ZF_LIB=str(lib))
    res = subprocess.run(
        [sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
         "tests/test_gpu_production.py", "tests/test_gpu_stats.py",
         "-k", "not checked and not one_wave"],
        cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-2000:]
    assert " passed" in res.stdout

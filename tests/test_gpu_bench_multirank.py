"""bench.py's N > 1 path (torchrun, max over ranks, allreduced validation and
config-5 counts, per-rank e2e, rank-0-only reference arm) run end to end with
two ranks sharing the one GPU of the test box over gloo
(ZF_BENCH_SHARE_DEVICE=1).  This checks the multi-rank code path, not
scaling: two ranks on one GPU measure nothing about 2 GPUs."""
import json
import os
import pathlib
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = pathlib.Path(__file__).resolve().parents[1]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _torchrun(args, timeout=600):
    env = dict(os.environ, ZF_BENCH_SHARE_DEVICE="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           str(ROOT / "bench.py"), "--gpus", "2", *args]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True,
                         timeout=timeout)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]  # rank 0 alone prints
    return lines[0]


def test_bench_two_ranks(cuda):
    n = 1 << 24
    d = _torchrun(["--steps", "2", "--warmup", "1", "--n-per-gpu", str(n), "--c5-total", str(1 << 30),
                   "--e2e-n", str(1 << 22), "--no-cpu-baseline"])
    assert d["n_gpus"] == 2 and d["steps"] == 2 and d["warmup"] == 1
    assert d["value"] == pytest.approx(2 * n / (d["ms_per_step"] * 1e-3))  # whole-job aggregate
    assert d["validation"]["allreduce"] == "gloo"  # (NCCL on a real multi-GPU node)
    assert d["validation"]["n_total"] == 2 * n and d["validation"]["passed"]
    assert d["c5"]["n_total_per_dist"] == 1 << 30 and d["c5"]["passed"]
    assert d["e2e"]["value"] > 0 and d["e2e"]["d2h_bytes_per_step"] == 8 * (1 << 22)
    assert "cpu_baseline" not in d
    assert d["gpu_launches"] == 2


def test_reference_arm_rank0_only(cuda):
    d = _torchrun(["--impl", "reference", "--steps", "1", "--warmup", "1", "--n-per-gpu", str(1 << 20)])
    assert d["impl"] == "reference" and d["n_gpus"] == 2
    assert d["e2e"]["value"] == d["value"] > 0

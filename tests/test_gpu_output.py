"""Output formats: the device '%.17g' formatter is
byte-identical to CPython's f"{v:.17g}" (the reference's `gen --format text`,
cli.py:100-120), and `gen` mirrors the reference CLI's behaviour."""
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def zf(cuda):
    import paper_1403_6870_b200 as zf
    return zf


def py_text(vals) -> bytes:
    return "".join(f"{v:.17g}\n" for v in np.asarray(vals, dtype=np.float64).tolist()).encode()


def device_text(zf, vals, cuda) -> bytes:
    import torch
    from paper_1403_6870_b200.output import format_g17
    t = torch.from_numpy(np.ascontiguousarray(vals, dtype=np.float64)).to(cuda)
    return format_g17(t).cpu().numpy().tobytes()


def test_edge_values(zf, cuda):
    vals = [0.0, -0.0, 1.0, -1.0, 0.1, 0.5, 1e-5, 1e-4, 9.999999999999999e-05, 0.0001,
            1e16, 1e16 - 2, 99999999999999984.0, 1e-22, 1.0000000000000001e-22,
            123.5, 1e15 + 0.5, 2.0 ** 52, 2.0 ** 53 - 1, 2.0 ** 56, 7.569274694148063,
            3.6360066255009458, 5e-324 * 0 + 2.2250738585072014e-20, 0.30000000000000004,
            1 / 3, 2 / 3, 1e-5 * 3, 12345678901234567.0, 9.5, 0.95, 0.095, 1.7976e16]
    vals += [np.nextafter(v, np.inf) for v in vals if 0 < v < 1e16]
    vals += [-v for v in vals]
    assert device_text(zf, vals, cuda) == py_text(vals)


def test_random_doubles_across_the_domain(zf, cuda):
    rng = np.random.default_rng(5)
    n = 1_000_000
    # log-uniform magnitudes in [1e-22, 1e17), random signs, plus random bit
    # patterns restricted to the domain
    mags = 10.0 ** rng.uniform(-22, 17, n)
    vals = np.where(rng.random(n) < 0.5, -mags, mags)
    bits = rng.integers(0, 2**63, n, dtype=np.uint64).view(np.float64)
    bits = bits[(np.abs(bits) >= 1e-22) & (np.abs(bits) < 1e17)]
    vals = np.concatenate([vals, bits, np.round(mags[:10000])])
    assert device_text(zf, vals, cuda) == py_text(vals)


@pytest.mark.parametrize("cls", ["ExpSampler", "NormalSampler", "TraditionalNormalSampler"])
def test_sampler_outputs(zf, cuda, cls):
    s = getattr(zf, cls)(source=zf.UniformSource.counter(3), device=cuda)
    vals = s.fill(500_000)
    from paper_1403_6870_b200.output import format_g17
    assert format_g17(vals).cpu().numpy().tobytes() == py_text(vals.cpu().numpy())


def test_unsupported_values_are_reported(zf, cuda):
    import torch
    from paper_1403_6870_b200.output import format_g17
    for bad in (1e17, 1e-23, float("inf"), float("nan")):
        with pytest.raises(ValueError):
            format_g17(torch.tensor([1.0, bad], dtype=torch.float64, device=cuda))
    assert format_g17(torch.empty(0, dtype=torch.float64, device=cuda)).numel() == 0


def run_gen(*args):
    return subprocess.run([sys.executable, "-m", "paper_1403_6870_b200.gen", *args],
                          capture_output=True)


def test_gen_matches_reference_behaviour(zf, orc, tmp_path):
    """reference tests/test_cli.py:62-102, 156-162"""
    out = run_gen("-n", "3", "--seed", "7")
    assert out.returncode == 0
    assert float(out.stdout.split()[0]) == 0.15069938164952687
    t, b = tmp_path / "v.txt", tmp_path / "v.bin"
    assert run_gen("--dist", "normal", "-n", "3000", "--seed", "9", "--out", str(t)).returncode == 0
    assert run_gen("--dist", "normal", "-n", "3000", "--seed", "9", "--format", "f64le",
                   "--out", str(b)).returncode == 0
    bin_vals = np.frombuffer(b.read_bytes(), dtype="<f8")
    want, _, _, _ = orc.fill_stream("normal", 3000, seed=9)
    assert np.array_equal(bin_vals.view(np.uint64), want.view(np.uint64))
    assert t.read_bytes() == py_text(want)
    z = tmp_path / "z.txt"
    assert run_gen("-n", "0", "--seed", "1", "--out", str(z)).returncode == 0
    assert z.read_bytes() == b""
    assert run_gen("-n", "-5", "--seed", "1").returncode == 2

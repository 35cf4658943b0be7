"""The C-ABI used from C (no Python in the sampling path): the library's
embedded default tables plus zf_fill, as a cgo / JNI / C host would call them."""
import pathlib
import subprocess

import numpy as np
import pytest

from helpers import assert_trad_close, bits

ROOT = pathlib.Path(__file__).resolve().parents[1]
SRC = ROOT / "tests" / "c" / "fill_default.c"
EXE = ROOT / "build" / "fill_default"
CUDA = pathlib.Path("/usr/local/cuda")


def compile_host(built_lib):
    EXE.parent.mkdir(parents=True, exist_ok=True)
    libdir = ROOT / "paper_1403_6870_b200"
    cmd = ["gcc", "-O2", "-std=c11", "-Wall", "-Werror", "-I", str(ROOT / "include"),
           "-I", str(CUDA / "include"), str(SRC), "-o", str(EXE),
           "-L", str(libdir), "-l:libzigfast_b200.so", "-L", str(CUDA / "lib64"), "-lcudart",
           f"-Wl,-rpath,{libdir}", f"-Wl,-rpath,{CUDA / 'lib64'}"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return EXE


def test_c_host_compiles_and_links(built_lib):
    assert compile_host(built_lib).exists()


@pytest.mark.gpu
@pytest.mark.parametrize("dist,name", [(0, "exp"), (1, "normal"), (2, "trad_exp"),
                                       (3, "trad_normal")])
def test_c_host_fill_matches_oracle(built_lib, orc, cuda, tmp_path, dist, name):
    exe = compile_host(built_lib)
    out = tmp_path / "v.bin"
    n, seed, base = 100_003, 99, 1 << 40
    subprocess.run([str(exe), str(dist), str(n), str(seed), str(base), str(out)], check=True,
                   timeout=120)
    got = np.fromfile(out, dtype="<f8")
    want, _, recs = orc.fill_ctr(name, n, seed=seed, ctr_base=base, records=True)
    assert_trad_close(got, bits(want), recs["path"] == 2, name)

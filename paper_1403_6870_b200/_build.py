"""Build the sm_100a shared library in-tree (libzigfast_b200.so next to this file).

nvcc cross-compiles for sm_100a without a GPU; the .so is git-ignored but
travels to the GPU box with the gpurun snapshot.  Used by __graft_entry__.build().
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import pathlib
import shutil
import subprocess

PKG = pathlib.Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = ROOT / "build" / "obj"
LIB = PKG / "libzigfast_b200.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
              "-I", str(ROOT / "include"), "-Xptxas", "-v"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and pathlib.Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cpp")))


def _compile(src: pathlib.Path, obj_dir: pathlib.Path = OBJ,
             extra: tuple = ()) -> tuple[pathlib.Path, str]:
    obj = obj_dir / (src.name + ".o")
    cmd = [nvcc(), *ARCH, *NVCC_FLAGS, *extra, "-c", str(src), "-o", str(obj)]
    if src.suffix == ".cpp":
        cmd = [nvcc(), *ARCH, "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-I",
               str(ROOT / "include"), "-c", str(src), "-o", str(obj)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src.name}:\n{res.stdout}\n{res.stderr}")
    return obj, res.stderr


def build(verbose: bool = False) -> pathlib.Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    srcs = sources()
    newest = max(p.stat().st_mtime for p in srcs + list(CSRC.glob("*.cuh")) +
                 list(CSRC.glob("*.h")) + list((ROOT / "include").glob("*.h")))
    if LIB.exists() and LIB.stat().st_mtime >= newest and not os.environ.get("ZF_REBUILD"):
        return LIB
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        results = list(ex.map(_compile, srcs))
    log = "\n".join(err for _, err in results)
    (ROOT / "build" / "ptxas.log").write_text(log)
    if verbose:
        print(log)
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc(), *ARCH, "-shared", "-o", str(tmp), *[str(o) for o, _ in results]]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stdout}\n{res.stderr}")
    os.replace(tmp, LIB)
    return LIB


def build_variant(name: str, defines: list[str]) -> pathlib.Path:
    """Experiment builds (e.g. -DZF_MIN_BLOCKS=6) into build/variants/<name>.so;
    select one at run time with ZF_LIB=<path>."""
    out_dir = ROOT / "build" / "variants"
    obj_dir = ROOT / "build" / f"obj_{name}"
    obj_dir.mkdir(parents=True, exist_ok=True)
    out_dir.mkdir(parents=True, exist_ok=True)
    extra = tuple(f"-D{d}" for d in defines)
    with cf.ThreadPoolExecutor(max_workers=8) as ex:
        results = list(ex.map(lambda s: _compile(s, obj_dir, extra), sources()))
    lib = out_dir / f"{name}.so"
    subprocess.run([nvcc(), *ARCH, "-shared", "-o", str(lib), *[str(o) for o, _ in results]],
                   check=True)
    return lib


if __name__ == "__main__":
    print(build(verbose=True))

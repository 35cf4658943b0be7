"""Run the fast-path micro-benchmarks (tools/ubench.cu) over grid sizes.

    python tools/ubench.py [log2 n]
"""
import ctypes as C
import pathlib
import subprocess
import sys

HERE = pathlib.Path(__file__).resolve().parent
SO = HERE / "_build" / "libubench.so"


def build():
    SO.parent.mkdir(exist_ok=True)
    if not SO.exists() or SO.stat().st_mtime < (HERE / "ubench.cu").stat().st_mtime:
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
                        "-Xcompiler", "-fPIC", "-shared", "-o", str(SO), str(HERE / "ubench.cu")],
                       check=True)


def main():
    build()
    import torch
    lib = C.CDLL(str(SO))
    lib.ub_run.argtypes = [C.c_int, C.c_void_p, C.c_uint64, C.c_void_p, C.c_int, C.c_void_p]
    n = 1 << int(sys.argv[1] if len(sys.argv) > 1 else 28)
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    tab = torch.rand(258, dtype=torch.float64, device="cuda") * 1e-19
    stream = torch.cuda.current_stream().cuda_stream
    for var in [int(a) for a in sys.argv[2].split(",")] if len(sys.argv) > 2 else range(8):
        for grid in (148 * 4, 148 * 16):
            for _ in range(3):
                lib.ub_run(var, out.data_ptr(), n, tab.data_ptr(), grid, stream)
            torch.cuda.synchronize()
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record()
            for _ in range(10):
                lib.ub_run(var, out.data_ptr(), n, tab.data_ptr(), grid, stream)
            t1.record()
            torch.cuda.synchronize()
            ms = t0.elapsed_time(t1) / 10
            print(f"v{var} grid {grid:5d}: {ms:.4f} ms  {n / ms / 1e6:7.1f} G/s  "
                  f"{8 * n / ms / 1e6:7.1f} GB/s", flush=True)


if __name__ == "__main__":
    main()

"""Whole-output parity sweep (evidence tool, not product): 2^32-sample production
fills, one launch each, every sample compared bit for bit with the CPU oracle
(`oracle.check_ctr`), over seeds, counter ranges up to the 2^44 limit and both
distributions; plus config 5 in full (2^36 + 2^36 draws counted on the device
vs `oracle.count_ctr`) with --c5.

    python tools/parity_sweep.py [--log2n 32] [--c5] > gpurun_out/r02d_full_parity.jsonl
"""
import argparse
import json
import pathlib
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log2n", type=int, default=32)
    ap.add_argument("--c5", action="store_true")
    a = ap.parse_args()
    import torch

    import paper_1403_6870_b200 as zf
    from oracle import oracle as orc
    from test_gpu_full_parity import _check_whole
    orc.build()
    dev = torch.device("cuda", 0)
    n = 1 << a.log2n
    total = 0
    cases = [(d, "f64", seed, base) for seed in (7, 99, 1234)
             for base in (0, 1 << 40, 7 << 40, (1 << 44) - n - 77) for d in ("normal", "exp")]
    cases += [(d, "f32", 7, 5 << 40) for d in ("normal", "exp")]
    for dist, dtype, seed, base in cases:
        m = n + 77
        t = time.time()
        bad, first = _check_whole(zf, orc, dev, dist, dtype, m, seed, base)
        total += m
        print(json.dumps({"dist": dist, "dtype": dtype, "seed": seed, "ctr_base": base, "n": m,
                          "mismatches": bad, "first": first,
                          "seconds": round(time.time() - t, 2)}), flush=True)
    print(json.dumps({"samples_compared": total}), flush=True)
    if a.c5:
        from paper_1403_6870_b200 import scale
        from paper_1403_6870_b200.tables import default_tables
        x1 = float(default_tables("exponential").x[1])
        m = 1 << 36
        t = time.time()
        got = ([int(c) for c in scale.device_counts("normal", scale.C5_SEED, 0, m,
                                                    scale.C5_THRESH, True, device=dev)] +
               [int(c) for c in scale.device_counts("exp", scale.C5_SEED, 0, m, (x1,), False,
                                                    device=dev)])
        t_dev = time.time() - t
        t = time.time()
        want = (orc.count_ctr("normal", m, scale.C5_SEED, 0, scale.C5_THRESH, True) +
                orc.count_ctr("exp", m, scale.C5_SEED, 0, (x1,), False))
        print(json.dumps({"config5_one_gpu": {"draws_per_dist": m, "device_counts": got,
                                              "oracle_counts": want, "equal": got == want,
                                              "device_s": round(t_dev, 2),
                                              "oracle_s": round(time.time() - t, 1)}}), flush=True)


if __name__ == "__main__":
    main()

"""Production-stream quality at scale (validation tooling): 2^k draws per
distribution and seed through the fused statistics kernel (nothing written),
raw moments 1..5 against the exact values (the reference's quality gate,
quality.py:24-42: |z| <= 6), a 1024-bin chi-square against the exact CDF, and
tail counts against the binomial mass.

    python tools/quality_at_scale.py [log2 n] [seeds...]
"""
import json
import math
import sys

import numpy as np

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1403_6870_b200 as zf  # noqa: E402
from paper_1403_6870_b200 import quality  # noqa: E402


def exp_cdf(x):
    return np.where(x > 0, -np.expm1(-np.maximum(x, 0.0)), 0.0)


def main():
    k = int(sys.argv[1]) if len(sys.argv) > 1 else 36
    seeds = [int(s) for s in sys.argv[2:]] or [7, 99]
    n = 1 << k
    dev = torch.device("cuda", 0)
    for dist, cls, lo, hi, th, cdf, absth in (
            ("normal", zf.NormalSampler, -6.0, 6.0, (5.0, 6.0, 7.0), quality.normal_cdf, True),
            ("exp", zf.ExpSampler, 0.0, 16.0, (7.569274694148063, 10.0, 15.0), exp_cdf, False)):
        for seed in seeds:
            s = cls(source=zf.UniformSource.counter(seed), device=dev)
            sums, res = quality.device_sums(s, n, moments=5, hist=(lo, hi, 1024), thresholds=th,
                                            abs_thresh=absth)
            raw = [v / n for v in sums]
            z = [(m - e) / (sd / math.sqrt(n)) for m, e, sd in
                 zip(raw, quality.EXPECTED_MOMENTS[dist], quality._MOMENT_SD[dist])]
            hist = np.asarray(res.hist)
            chi2, dof, chi2_z = quality.histogram_chi2(hist, n, lo, hi, cdf=cdf)
            tails = []
            for t, c in zip(th, res.thresh_counts):
                p = math.erfc(t / math.sqrt(2.0)) if dist == "normal" else math.exp(-t)
                ok, mu, sd = quality.binomial_check(int(c), n, p)
                tails.append({"gt": t, "count": int(c), "expected": mu, "sd": sd, "within_5sigma": ok})
            print(json.dumps({"dist": dist, "seed": seed, "n": n, "raw_moment_z": z,
                              "hist_chi2": chi2, "hist_dof": dof, "hist_z": chi2_z, "tails": tails,
                              "passed": all(abs(v) <= 6 for v in z) and abs(chi2_z) <= 6
                              and all(t["within_5sigma"] for t in tails)}), flush=True)


if __name__ == "__main__":
    main()

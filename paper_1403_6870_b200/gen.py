"""`gen` entry point: stream variates to stdout or a file, as the reference's
`zigfast gen` does (`cli.py:45-50, 100-120`): same options, same bytes, exit
codes 0 (ok) / 2 (operational failure).  The rest of the reference's CLI
(tables, quality, bench, pathstats) is out of scope.

    python -m paper_1403_6870_b200.gen --dist exp -n 1000 --seed 7 [--format text|f64le]
        [--out PATH] [--generator xoshiro256++|splitmix64|ctr] [--traditional]

`--seed` wins over ZIGFAST_SEED, which wins over auto-seeding (uniform.py:48-60).
The default generator is the reference's xoshiro256++ (oracle mode, identical
values); `--generator ctr` selects the production counter stream.
"""

from __future__ import annotations

import argparse
import sys

OK, OP_FAIL = 0, 2


def _parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_1403_6870_b200.gen")
    ap.add_argument("--dist", choices=("exp", "normal"), default="exp")
    ap.add_argument("-n", type=int, required=True)
    ap.add_argument("--seed", type=int, default=None)
    ap.add_argument("--format", choices=("text", "f64le"), default="text")
    ap.add_argument("--out", default=None)
    ap.add_argument("--generator", choices=("xoshiro256++", "splitmix64", "ctr"),
                    default="xoshiro256++")
    ap.add_argument("--traditional", action="store_true",
                    help="the traditional ziggurat baseline instead of the modified one")
    return ap


def main(argv=None) -> int:
    args = _parser().parse_args(argv)
    if args.n < 0:
        print("n must be >= 0", file=sys.stderr)
        return OP_FAIL
    import paper_1403_6870_b200 as zf
    from .output import write_values
    try:
        src = (zf.UniformSource.counter(args.seed) if args.generator == "ctr"
               else zf.UniformSource(args.seed, args.generator))
        if args.traditional:
            cls = zf.TraditionalExpSampler if args.dist == "exp" else zf.TraditionalNormalSampler
        else:
            cls = zf.ExpSampler if args.dist == "exp" else zf.NormalSampler
        sampler = cls(source=src)
        sink = open(args.out, "wb") if args.out else sys.stdout.buffer
        try:
            write_values(sampler, args.n, sink, args.format, chunk=1 << 20)
        finally:
            if args.out:
                sink.close()
    except (zf.ZigfastError, OSError, ValueError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return OP_FAIL
    return OK


if __name__ == "__main__":
    sys.exit(main())

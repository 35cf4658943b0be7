"""Basic-block summary of an ncu report's SASS source page (experiment tool).

    python tools/ncu_blocks.py report.ncu-rep [min_share]

Prints runs of consecutive SASS instructions with the same execution count
(one basic block each) with their share of executed instructions and of
warp-stall samples, and the most common opcodes."""
import collections
import csv
import io
import subprocess
import sys

path = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.002
txt = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[1]
data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
IE, ST = ix["Instructions Executed"], ix["Warp Stall Sampling (All Samples)"]
TH = ix["Avg. Threads Executed"]
tot_i = sum(int(r[IE]) for r in data)
tot_s = sum(int(r[ST]) for r in data)
print(f"instructions {tot_i}, stall samples {tot_s}")


def op(s):
    t = s.strip().split()
    return (t[1] if t[0].startswith("@") else t[0]).split(".")[0]


blocks, cur = [], None
for k, r in enumerate(data):
    ie, st = int(r[IE]), int(r[ST])
    if ie == 0 and st == 0:
        cur = None
        continue
    if cur and cur["ie"] == ie:
        cur["n"] += 1
        cur["st"] += st
        cur["end"] = k
        cur["ops"].append(op(r[1]))
    else:
        cur = dict(start=k, end=k, ie=ie, n=1, st=st, ops=[op(r[1])], thr=float(r[TH]))
        blocks.append(cur)
for b in blocks:
    fi, fs = b["ie"] * b["n"] / tot_i, b["st"] / tot_s
    if fi > thr or fs > thr:
        c = collections.Counter(b["ops"]).most_common(6)
        print(f"{b['start']:5d}-{b['end']:5d} n={b['n']:4d} exec={b['ie']:9d} inst%={fi*100:5.2f} "
              f"stall%={fs*100:5.2f} thr={b['thr']:4.1f} {dict(c)}")

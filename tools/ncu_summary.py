"""Summarise an ncu report (raw page): key metrics for the profiled kernel(s).

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [more.ncu-rep ...]
"""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "sm__cycles_elapsed.avg.per_second",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
]


def summary(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]
    out = []
    for row in rows[2:]:
        name = row[head.index("Kernel Name")] if "Kernel Name" in head else "?"
        d = {"kernel": name[:90]}
        for k in KEYS:
            if k in head:
                i = head.index(k)
                d[k] = f"{row[i]} {units[i]}".strip()
        stalls = {}
        for i, h in enumerate(head):
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    stalls[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(row[i])
                except ValueError:
                    pass
        tot = sum(stalls.values()) or 1.0
        d["stall_top"] = ", ".join(f"{k} {v / tot:.0%}" for k, v in
                                   sorted(stalls.items(), key=lambda kv: -kv[1])[:6])
        out.append(d)
    return out


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print("==", p)
        for d in summary(p):
            for k, v in d.items():
                print(f"  {k}: {v}")

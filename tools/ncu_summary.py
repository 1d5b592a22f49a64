"""Compact per-kernel summary of an ncu report (--page raw --csv) or a launch-list CSV.

  python tools/ncu_summary.py report.ncu-rep        # full-set metrics + top stall reasons
  python tools/ncu_summary.py --launches launches.csv
"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%peak"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma_pipe_%"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64_pipe_%"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_pipe_%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__block_size", "block"),
    ("launch__grid_size", "grid"),
    ("launch__occupancy_limit_registers", "occ_lim_regs"),
    ("launch__occupancy_limit_shared_mem", "occ_lim_smem"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_bank_conflicts"),
    ("smsp__inst_executed.sum", "inst_executed"),
]


def short(name):
    name = re.sub(r"\(.*", "", name)
    name = name.replace("(anonymous namespace)::", "").replace("erxk::", "").replace("void ", "")
    return name.strip()


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    units = rows[1]
    for r in rows[2:]:
        d = dict(zip(h, r))
        print(f"== {short(d.get('Kernel Name', '?'))}")
        for key, label in KEYS:
            if key in d:
                u = units[h.index(key)]
                print(f"   {label:22s} {d[key]} {u}")
        st = []
        for i, k in enumerate(h):
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                try:
                    st.append((k[len("smsp__pcsamp_warps_issue_stalled_"):], float(r[i].replace(",", ""))))
                except ValueError:
                    pass
        tot = sum(v for _, v in st) or 1.0
        st.sort(key=lambda x: -x[1])
        print("   stalls:", ", ".join(f"{k}={v / tot:.2f}" for k, v in st[:6]))


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    t = defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            t[short(r[ki])].append(float(r[vi].replace(",", "")))
    ours = {k: v for k, v in t.items() if any(s in k for s in ("stats", "scan", "factor", "score", "normalize"))}
    tot = sum(sum(v) for v in ours.values()) or 1.0
    print(f"{'kernel':34s} {'launches':>8s} {'mean':>12s} {'share':>6s}")
    for k, v in sorted(ours.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k:34s} {len(v):8d} {sum(v) / len(v):12.1f} {sum(v) / tot:6.3f}")
    print("(ns; ncu --clock-control none, serialised cold-cache launches: compare shares, not absolutes)")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2])
    else:
        full(sys.argv[1])

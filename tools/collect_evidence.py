"""Copy one evidence pass from gpurun_out/ (scratch) into profiles/ (tracked):
  python tools/collect_evidence.py r02e
bench / reference JSON lines, GPU test tail, parity table, the launch list (per-kernel mean and share from
the ncu gpu__time_duration pass) and tools/ncu_summary.py summaries of the --set full captures."""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
tag = sys.argv[1]


def copy(src, dst):
    sp = os.path.join(G, src)
    if os.path.exists(sp):
        open(os.path.join(P, dst), "w").write(open(sp).read())
        print("wrote", dst)


def last_json_line(path):
    for line in reversed(open(path).read().splitlines()):
        if line.startswith("{"):
            return line
    return None


for src, dst in ((f"bench_{tag}.json", f"{tag}_bench.json"), (f"ref_{tag}.json", f"{tag}_bench_reference.json")):
    sp = os.path.join(G, src)
    if os.path.exists(sp):
        line = last_json_line(sp)
        if line:
            open(os.path.join(P, dst), "w").write(line + "\n")
            print("wrote", dst)
copy(f"parity_{tag}.jsonl", f"{tag}_parity_fullstream.jsonl")
copy(f"launches_{tag}.csv", f"{tag}_launches.csv")
copy(f"kt_{tag}.log", f"{tag}_kernel_times.txt")
sp = os.path.join(G, f"gputests_{tag}.log")
if os.path.exists(sp):
    open(os.path.join(P, f"{tag}_gputests_tail.txt"), "w").write("\n".join(open(sp).read().splitlines()[-6:]) + "\n")
    print("wrote gputests tail")
sp = os.path.join(G, f"launches_{tag}.csv")
if os.path.exists(sp):
    rows = [r for r in csv.reader(l for l in open(sp) if not l.startswith("=="))]
    hdr = next((r for r in rows if "Kernel Name" in r), None)
    if hdr:
        ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
        acc = defaultdict(list)
        for r in rows[rows.index(hdr) + 1:]:
            if len(r) > vi and r[vi].replace(",", "").replace(".", "").isdigit():
                acc[r[ki]].append(float(r[vi].replace(",", "")))
        tot = sum(sum(v) for v in acc.values()) or 1.0
        with open(os.path.join(P, f"{tag}_launches.txt"), "w") as f:
            f.write(f"{'kernel':<60s} {'launches':>8s} {'mean':>12s} {'share':>6s}\n")
            for k, v in sorted(acc.items(), key=lambda kv: -sum(kv[1])):
                f.write(f"{k[:60]:<60s} {len(v):8d} {sum(v) / len(v):12.1f} {sum(v) / tot:6.3f}\n")
            f.write("(ns; ncu --clock-control none, serialised cold-cache launches: compare shares, not absolutes;\n"
                    " at:: kernels are torch's input-pool setup and checks outside the timed region)\n")
        print("wrote launch list")
for rep, dst in ((f"{tag}_c3.ncu-rep", f"{tag}_ncu_full_c3.txt"), (f"{tag}_c3srp.ncu-rep", f"{tag}_ncu_full_c3srp.txt"),
                 (f"{tag}_c2.ncu-rep", f"{tag}_ncu_full_c2.txt")):
    sp = os.path.join(G, rep)
    if os.path.exists(sp):
        out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), sp], capture_output=True,
                             text=True).stdout
        open(os.path.join(P, dst), "w").write(out)
        print("wrote", dst)

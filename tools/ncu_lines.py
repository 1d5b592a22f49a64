"""Per-source-line stall samples / executed instructions from `ncu -i R --page source --csv --print-source cuda,sass`.

  ncu -i rep.ncu-rep [-k regex:NAME] --page source --csv --print-source cuda,sass > x.csv
  python tools/ncu_lines.py x.csv [top]
"""
import csv
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    fname = "?"
    out = []
    hdr = None
    for r in csv.reader(open(path)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] in ("Function Name",) or not r[0].isdigit():
            continue
        d = dict(zip(hdr[2:], r[2:]))
        if r[2] != "-":
            continue  # sass rows under the cuda line
        try:
            s = float(d["Warp Stall Sampling (All Samples)"] or 0)
            n = float(d["Instructions Executed"] or 0)
        except (KeyError, ValueError):
            continue
        out.append((s, n, fname, int(r[0]), r[1][:90]))
    ts = sum(o[0] for o in out) or 1
    tn = sum(o[1] for o in out) or 1
    print(f"samples {ts:.0f}  warp-instructions {tn:.0f}")
    for s, n, f, ln, src in sorted(out, reverse=True)[:top]:
        print(f"{100 * s / ts:5.1f}% stall {100 * n / tn:5.1f}% inst  {f}:{ln}  {src.strip()}")


if __name__ == "__main__":
    main()

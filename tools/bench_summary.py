"""Print the key numbers of bench.py JSON lines (files given on argv)."""
import json
import sys

for path in sys.argv[1:]:
    lines = [x for x in open(path) if x.startswith("{")]
    if not lines:
        print(path, "NO JSON:", open(path).read()[-800:])
        continue
    d = json.loads(lines[-1])
    e2e = d.get("e2e") or {}
    print(f"{path}: value={d['value']:.0f} {d['unit']} e2e={e2e.get('value', 0):.0f} "
          f"factor={d['config'].get('factor_precision')} T={d['config'].get('window_lines')} "
          f"roof[{d['roofline']['kernel']}]={d['roofline']['frac']:.3f} line_frac={d['roofline_line']['frac']:.3f} "
          f"clk={d['clocks'].get('sm_mhz')}")
    for k, v in d["kernels"].items():
        tf = v.get("tflops")
        print(f"   {k:10s} {v['ms_per_launch']:.3f} ms  share {v['share']:.3f}  {tf and round(tf, 2)} TF/s")
    for k in ("single_stream", "single_stream_c2", "batched_srp", "batched_c4", "latency"):
        if k in d:
            print("  ", k, json.dumps(d[k])[:300])

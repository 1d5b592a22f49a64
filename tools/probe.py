"""Measure FFMA / FFMA2 throughput on the current GPU (prints JSON; liberx_probe.so)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_14947_b200 import probe  # noqa: E402

r, c = probe.fp32_tflops()
print(json.dumps({"ffma_reg_tflops": r, "ffma_const_tflops": c, "ffma2_reg_tflops": probe.ffma2_tflops()}))

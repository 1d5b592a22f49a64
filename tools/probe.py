"""Measure FFMA / FFMA2 throughput on the current GPU (prints JSON)."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_14947_b200 as pkg

eng = pkg.Engine(pkg.ErxConfig(no_srp=True), 8)
r, c = eng.probe_fp32_tflops()
f2 = C.c_double(0)
pkg.lib().erx_probe_ffma2_tflops(eng._h, C.byref(f2))
print(json.dumps({"ffma_reg_tflops": r, "ffma_const_tflops": c, "ffma2_reg_tflops": f2.value}))

"""Measure global->shared streaming paths on this GPU (erx_probe_stream, liberx_probe.so).

  python tools/stream_probe.py            # HBM-sized buffer (1 GiB) and L2-resident buffer (48 MiB)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_14947_b200 import probe  # noqa: E402

for size, label in ((1 << 30, "HBM 1GiB"), (48 << 20, "L2 48MiB")):
    for mode, chunk, stages, cps in [(1, 32768, 1, 2), (0, 27648, 4, 1), (0, 27648, 2, 1), (0, 65536, 3, 1),
                                     (0, 16384, 4, 2), (2, 27648, 4, 1)]:
        g = probe.stream_gbs(mode, chunk, stages, cps, size)
        print(f"{label} mode {mode} chunk {chunk:6d} stages {stages} ctas/SM {cps}: {g:8.1f} GB/s")

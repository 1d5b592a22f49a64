#!/bin/bash
# source-level ncu captures of the configs[3] pipeline kernels (one launch each)
python tools/kt_probe.py 3 full 0 3 > gpurun_out/plain_c3.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"${1:-stats_i8_kernel|factor_blk|score_i8_kernel|scan_kernel}" \
    -s 4 -c ${2:-4} -o gpurun_out/src_c3 python tools/kt_probe.py 3 full 0 3 > gpurun_out/ncu_src.log 2>&1
echo ncu rc=$?

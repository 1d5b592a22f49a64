ncu --set full --clock-control none --import-source on -k regex:"stats_small|score_small" \
    -s 4 -c 2 -o gpurun_out/r02e_c2wl python tools/kt_probe.py 2 full 2048 3 > gpurun_out/ncu_c2wl.log 2>&1
echo ncu rc=$?

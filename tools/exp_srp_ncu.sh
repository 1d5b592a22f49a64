ncu --set full --clock-control none --import-source on -k regex:"stats_small_srp" \
    -s 2 -c 1 -o gpurun_out/r02e_c3srp env ERX_DEVICE_GROUPS=1 python tools/kt_probe.py 3 srp 32 3 > gpurun_out/ncu_c3srp.log 2>&1
echo ncu rc=$?

# round-2 ncu captures (one tool per call): c3 pipeline kernels, then the wide kernels of c1 / c4
python tools/kt_probe.py 3 full 0 3 > gpurun_out/plain_c3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"stats_i8_kernel|c0_fold|scan_kernel|factor_blk|score_i8_kernel|normalize|fixup" \
    -s 7 -c 7 -o gpurun_out/r02_c3 python tools/kt_probe.py 3 full 0 3 > gpurun_out/ncu_c3.log 2>&1
echo c3 rc=$?
python tools/kt_probe.py 1 full 256 3 > gpurun_out/plain_c1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"range_kernel|stats_i8t|wplanes|score_i8w|factor_blk" \
    -s 5 -c 5 -o gpurun_out/r02_c1 python tools/kt_probe.py 1 full 256 3 > gpurun_out/ncu_c1.log 2>&1
echo c1 rc=$?
ERX_FACTOR=30 python tools/kt_probe.py 4 full 32 2 > gpurun_out/plain_c4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"factor_cl|factor_big" -s 1 -c 1 \
    -o gpurun_out/r02_c4cl env ERX_FACTOR=30 python tools/kt_probe.py 4 full 32 2 > gpurun_out/ncu_c4.log 2>&1
echo c4 rc=$?

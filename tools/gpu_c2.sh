# configs[2] (10 bands, D <= 16 path): per-kernel times and an ncu --set full capture of its kernels
timeout 600 python -m pytest tests/test_gpu_numerics.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "radiance or onepass or split" 2>&1 | tail -3
python tools/kt_probe.py 2 full 2048 20 > gpurun_out/kt_c2.log 2>&1; python tools/kt_probe.py 2 srp 2048 20 >> gpurun_out/kt_c2.log 2>&1; cat gpurun_out/kt_c2.log
ncu --set full --clock-control none --import-source on -k regex:"stats_small|scan|factor|score_small|fixup" \
    -s 5 -c 5 -o gpurun_out/r02e_c2 python tools/kt_probe.py 2 full 2048 3 > gpurun_out/ncu_c2.log 2>&1
echo ncu rc=$?

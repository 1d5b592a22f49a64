# round-2 (second half) evidence run: full GPU tests with the parity log, bench, reference arm,
# launch list, ncu --set full of the configs[3] pipeline kernels
export ERX_PARITY_LOG=gpurun_out/parity_r02d.jsonl
rm -f $ERX_PARITY_LOG
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --tb=short > gpurun_out/gputests_r02d.log 2>&1
tail -3 gpurun_out/gputests_r02d.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02d.json 2> gpurun_out/bench_r02d.err; echo bench rc=$?
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref_r02d.json 2>&1; echo ref rc=$?
python bench.py --steps 2 --warmup 3 --quick --no-cpu > gpurun_out/plain_launch.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_r02d.csv \
    python bench.py --steps 2 --warmup 3 --quick --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?
ERX_DEVICE_GROUPS=1 python tools/kt_probe.py 3 full 0 3 > gpurun_out/plain_c3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"stats_i8_ws_kernel|stats_i8_kernel|c0_fold|scan_tile_kernel|scan_kernel|factor_blk|score_i8_kernel|normalize|fixup" \
    -s 7 -c 7 -o gpurun_out/r02d_c3 env ERX_DEVICE_GROUPS=1 python tools/kt_probe.py 3 full 0 3 > gpurun_out/ncu_c3.log 2>&1
echo ncu rc=$?

# round-2 evidence run (pass j, final): full GPU tests with the parity log, bench, reference arm,
# launch list, ncu --set full of the configs[3] pipeline (D = B, one 4096-line group per launch) and of the
# warp-per-line small-D kernels (configs[3] d = 5, configs[2])
export ERX_PARITY_LOG=gpurun_out/parity_r02j.jsonl
rm -f $ERX_PARITY_LOG
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --tb=short > gpurun_out/gputests_r02j.log 2>&1
tail -3 gpurun_out/gputests_r02j.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02j.json 2> gpurun_out/bench_r02j.err; echo bench rc=$?
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref_r02j.json 2>&1; echo ref rc=$?
python bench.py --steps 2 --warmup 3 --quick --no-cpu > gpurun_out/plain_launch.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches_r02j.csv \
    python bench.py --steps 2 --warmup 3 --quick --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?
ERX_DEVICE_GROUPS=1 python tools/kt_probe.py 3 full 64 3 > gpurun_out/plain_c3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"stats_i8_ws_kernel|stats_i8_kernel|c0_fold|scan_tile_kernel|scan_kernel|factor_blk|score_i8_kernel|normalize|fixup" \
    -s 7 -c 7 -o gpurun_out/r02j_c3 env ERX_DEVICE_GROUPS=1 python tools/kt_probe.py 3 full 64 3 > gpurun_out/ncu_c3.log 2>&1
echo ncu c3 rc=$?
ERX_DEVICE_GROUPS=1 python tools/kt_probe.py 3 srp 128 3 > gpurun_out/plain_c3srp.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"stats_small|scan|factor_blk|score_small|fixup" \
    -s 5 -c 5 -o gpurun_out/r02j_c3srp env ERX_DEVICE_GROUPS=1 python tools/kt_probe.py 3 srp 128 3 > gpurun_out/ncu_c3srp.log 2>&1
echo ncu c3srp rc=$?
python tools/kt_probe.py 2 full 2048 3 > gpurun_out/plain_c2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"stats_small|scan|factor_blk|score_small|fixup" \
    -s 5 -c 5 -o gpurun_out/r02j_c2 python tools/kt_probe.py 2 full 2048 3 > gpurun_out/ncu_c2.log 2>&1
echo ncu c2 rc=$?
for a in "3 full 64 20" "3 srp 128 20" "3 srp 64 20" "2 full 2048 20" "1 full 256 20" "4 full 32 10" "4 full 128 4" "1 full 1024 5" "0 full 32 20"; do python tools/kt_probe.py $a; done > gpurun_out/kt_r02j.log 2>&1
cat gpurun_out/kt_r02j.log

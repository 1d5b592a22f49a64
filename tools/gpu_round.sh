# one GPU round: parity tests, smoke, bench, ncu launch list + full captures of the top kernels
set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --quick > gpurun_out/bench_main.log 2>&1; echo "bench exit $?"
timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu --quick > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --steps 4 --warmup 3 --no-cpu --quick > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stats_kernel|score_kernel|factor_blk" -s 5 -c 3 -o gpurun_out/prof_r3 python bench.py --steps 4 --warmup 3 --no-cpu --quick > gpurun_out/ncu_full.log 2>&1; echo "ncu full exit $?"

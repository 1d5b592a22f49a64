# one GPU round: parity tests, smoke, full bench, ncu launch list + full captures of the top kernels
set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench exit $?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "ref exit $?"
timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu --quick > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 4 --warmup 3 --no-cpu --quick > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stats_i8|score_i8|factor_blk" -s 5 -c 3 -o gpurun_out/prof_round python bench.py --steps 4 --warmup 3 --no-cpu --quick > gpurun_out/ncu_full.log 2>&1; echo "ncu full exit $?"
timeout 300 python bench.py --config 4 --window 32 --steps 5 --warmup 3 --no-cpu --quick > gpurun_out/bench_c4.log 2>&1; echo "c4 exit $?"
timeout 300 python bench.py --config 1 --window 256 --steps 5 --warmup 3 --no-cpu --quick > gpurun_out/bench_c1.log 2>&1; echo "c1 exit $?"
python tools/ncu_summary.py gpurun_out/prof_round.ncu-rep > gpurun_out/ncu_full_summary.txt 2>&1
python tools/ncu_summary.py --launches gpurun_out/launches.csv > gpurun_out/launches_summary.txt 2>&1

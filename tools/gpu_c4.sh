cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --config 4 --window 32 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_c4.log 2>&1; echo "bench c4 exit $?"; python tools/bench_summary.py gpurun_out/bench_c4.log 2>/dev/null | head -8
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --quick > gpurun_out/bench_q.log 2>&1; echo "bench exit $?"; python tools/bench_summary.py gpurun_out/bench_q.log 2>/dev/null | head -9

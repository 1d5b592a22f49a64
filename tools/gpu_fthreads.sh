cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_gpu.log
for t in ${FT_LIST:-64 128 256}; do ERX_FACTOR_THREADS=$t timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --quick > gpurun_out/bench_ft$t.log 2>&1; echo "threads $t exit $?"; python tools/bench_summary.py gpurun_out/bench_ft$t.log | head -4; done

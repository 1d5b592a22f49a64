cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_gpu.log
for m in "" "--sync-host"; do timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --quick $m > gpurun_out/exp_e2e.log 2>&1; echo "e2e $m: $(python tools/bench_summary.py gpurun_out/exp_e2e.log 2>/dev/null | head -1)"; done

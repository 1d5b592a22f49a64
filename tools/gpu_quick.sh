# quick GPU check: parity tests (subset or all) + bench (no cpu baseline)
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --quick > gpurun_out/bench_q.log 2>&1; echo "bench exit $?"
python tools/bench_summary.py gpurun_out/bench_q.log
if [ -n "$NCU_K" ]; then
  timeout 900 ncu --set full --clock-control none -k regex:"$NCU_K" -s 2 -c 1 -o gpurun_out/prof_q python bench.py --steps 4 --warmup 3 --no-cpu --quick > gpurun_out/ncu_q.log 2>&1; echo "ncu exit $?"
  python tools/ncu_summary.py gpurun_out/prof_q.ncu-rep | grep -E "==|duration|dram_read|dram_write|tensor_pipe|issue_active"
fi

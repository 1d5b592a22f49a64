# GPU check of the drop-in host path: parity tests + bench e2e with 1 vs auto stream groups
set -x
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -5 gpurun_out/pytest_gpu.log
for g in 1 0 4 8; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --quick --host-groups $g > gpurun_out/bench_g$g.log 2>&1; echo "bench g$g exit $?"
  python tools/bench_summary.py gpurun_out/bench_g$g.log 2>/dev/null | head -3
done

# quick GPU check: parity tests + bench (no ncu)
set -x
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -5 gpurun_out/pytest_gpu.log
for f in 32 64; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --quick --factor $f > gpurun_out/bench_f$f.log 2>&1; echo "bench f$f exit $?"
done

# exact-int8 tcgen05 path: parity tests + bench comparison
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "stats" -s > gpurun_out/pytest_i8.log 2>&1; echo "pytest exit $?"
tail -2 gpurun_out/pytest_i8.log; grep "stats tensor" gpurun_out/pytest_i8.log
for k in 0 2; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --quick --stats $k > gpurun_out/bench_s$k.log 2>&1
  python tools/bench_summary.py gpurun_out/bench_s$k.log
done

# exact-int8 tcgen05 stats: parity tests + bench comparison + ring-depth experiments
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "stats" -s > gpurun_out/pytest_i8.log 2>&1; echo "pytest exit $?"
tail -3 gpurun_out/pytest_i8.log
for cfg in "0 0" "1 0" "0 4" "0 3"; do
  set -- $cfg
  ERX_I8_DEBUG=$1 ERX_I8_STAGES=$2 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --quick --stats 2 > gpurun_out/bench_x.log 2>&1
  echo "dbg $1 stages $2: $(python tools/bench_summary.py gpurun_out/bench_x.log 2>&1 | grep stats)"
done

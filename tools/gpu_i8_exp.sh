cd $GRAFT_REPO_ROOT
for t in 32 64 96 128; do
  ERX_FT=$t timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --quick > gpurun_out/bench_x.log 2>&1
  echo "threads $t: $(python tools/bench_summary.py gpurun_out/bench_x.log 2>&1 | grep ' factor ')"
done

# stats_i8 ablations: ERX_I8_DEBUG bit 1 no MMAs, 2 no quantisation, 4 no range pass, 8 no epilogue math
cd $GRAFT_REPO_ROOT
for d in 0 1 2 4 8 3 15; do
  ERX_I8_DEBUG=$d timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --quick > gpurun_out/bench_x.log 2>&1
  echo "dbg $d: $(python tools/bench_summary.py gpurun_out/bench_x.log 2>&1 | grep ' stats ')"
done

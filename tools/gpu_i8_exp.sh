# score_i8 ablations: ERX_I8_DEBUG bit 1 no MMAs, bit 2 no quantisation, bit 4 no epilogue math
cd $GRAFT_REPO_ROOT
for d in 0 1 2 4 6 7; do
  ERX_I8_DEBUG=$d timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --quick > gpurun_out/bench_x.log 2>&1
  echo "dbg $d: $(python tools/bench_summary.py gpurun_out/bench_x.log 2>&1 | grep " score ")"
done

# stats_i8 experiments: ERX_I8_DEBUG 0 normal, 1 no compute; ERX_I8_SPLIT copies per chunk; ERX_I8_STAGES ring depth
cd $GRAFT_REPO_ROOT
for cfg in "0 1 0" "1 1 0" "0 1 4" "0 1 3"; do
  set -- $cfg
  ERX_I8_DEBUG=$1 ERX_I8_SPLIT=$2 ERX_I8_STAGES=$3 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --quick --stats 2 > gpurun_out/bench_x.log 2>&1
  echo "dbg $1 split $2 stages $3: $(python tools/bench_summary.py gpurun_out/bench_x.log 2>&1 | grep stats)"
done

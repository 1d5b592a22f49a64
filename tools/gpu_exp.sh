cd $GRAFT_REPO_ROOT
run() { name=$1; shift; env "$@" timeout 300 python bench.py --config $CFG --window $WIN --steps 5 --warmup 3 --no-cpu --quick > gpurun_out/exp_$name.log 2>&1; echo "$name: $(python tools/bench_summary.py gpurun_out/exp_$name.log 2>/dev/null | head -5 | tr -s ' ' | tr '\n' '|')"; }
CFG=4 WIN=32
run c4_base X=1
run c4_nt256 ERX_STATS_NT=256
run c4_nt192 ERX_STATS_NT=192
CFG=1 WIN=256
run c1_nt256 ERX_STATS_NT=256 ERX_SCORE_WSMEM=0
run c1_nt192 ERX_STATS_NT=192 ERX_SCORE_WSMEM=0

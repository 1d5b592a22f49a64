cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_gpu.log
run() { name=$1; shift; env "$@" timeout 300 python bench.py --config $CFG --window $WIN --steps 5 --warmup 3 --no-cpu --quick > gpurun_out/exp_$name.log 2>&1; echo "$name: $(python tools/bench_summary.py gpurun_out/exp_$name.log 2>/dev/null | head -4 | tr -s ' ' | tr '\n' '|')"; }
CFG=1 WIN=256; run c1 X=1
CFG=3 WIN=32; run c3 X=1
CFG=0 WIN=32; run c0 X=1

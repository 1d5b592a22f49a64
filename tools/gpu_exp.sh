cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_gpu.log
run() { name=$1; shift; timeout 300 python bench.py "$@" --steps 5 --warmup 3 --no-cpu --quick > gpurun_out/exp_$name.log 2>&1; echo "$name: $(python tools/bench_summary.py gpurun_out/exp_$name.log 2>/dev/null | head -3 | tr -s ' ' | tr '\n' '|')"; }
run c3srp --config 3 --window 32 --mode srp
run c2_w256 --config 2 --window 256
run c2srp_w256 --config 2 --window 256 --mode srp

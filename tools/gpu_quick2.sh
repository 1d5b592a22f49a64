cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
for c in "3 full 16" "0 full 64" "1 full 64" "0 full 256"; do
  set -- $c
  timeout 600 python bench.py --config $1 --mode $2 --window $3 --steps 6 --warmup 2 --no-cpu --quick > gpurun_out/bench_c$1_$2_$3.log 2>&1; echo "c$1 $2 $3 exit $?"
done

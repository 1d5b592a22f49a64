# bench with each experiment env var of $EXPVARS set in turn (first run: none)
cd $GRAFT_REPO_ROOT
for v in none $EXPVARS; do
 ( if [ $v != none ]; then export $v=1; fi
 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --quick > gpurun_out/exp_$v.log 2>&1; echo "== $v"; python tools/bench_summary.py gpurun_out/exp_$v.log 2>/dev/null | head -3 )
done

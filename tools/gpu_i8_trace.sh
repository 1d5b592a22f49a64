cd $GRAFT_REPO_ROOT
ERX_I8_DEBUG=10 timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu --quick --stats 2 > gpurun_out/trace.log 2>&1
grep "score totals" gpurun_out/trace.log | head -4

cd $GRAFT_REPO_ROOT
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu --quick > gpurun_out/trace.log 2>&1
grep "factor line0" gpurun_out/trace.log | head -6

cd $GRAFT_REPO_ROOT
ERX_I8_DEBUG=32 timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu --quick > gpurun_out/trace.log 2>&1
grep "stats CTA0" gpurun_out/trace.log | head -4

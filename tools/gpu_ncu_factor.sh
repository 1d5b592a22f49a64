# ncu --set full of one factor_blk launch (threads from $ERX_FACTOR_THREADS, default heuristic)
cd $GRAFT_REPO_ROOT
timeout 300 python bench.py --steps 4 --warmup 3 --no-cpu --quick > gpurun_out/nf_plain.log 2>&1; echo "plain exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:factor_blk -s 2 -c 1 -o gpurun_out/prof_factor python bench.py --steps 4 --warmup 3 --no-cpu --quick > gpurun_out/ncu_factor.log 2>&1; echo "ncu exit $?"
python tools/ncu_summary.py gpurun_out/prof_factor.ncu-rep

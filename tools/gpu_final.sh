# round-end evidence: the gpu_round set plus ncu summaries of the side-workload kernels
cd $GRAFT_REPO_ROOT
bash tools/gpu_round.sh
timeout 600 ncu --set full --clock-control none -k regex:"stats_small|score_small" -s 4 -c 2 -o gpurun_out/prof_srp python bench.py --config 3 --mode srp --steps 4 --warmup 3 --no-cpu --quick > gpurun_out/ncu_srp.log 2>&1; echo "ncu srp exit $?"
timeout 600 ncu --set full --clock-control none -k regex:"stats_kernel|score_kernel|factor_blk" -s 9 -c 3 -o gpurun_out/prof_c1 python bench.py --config 1 --window 256 --steps 4 --warmup 3 --no-cpu --quick > gpurun_out/ncu_c1.log 2>&1; echo "ncu c1 exit $?"
timeout 600 ncu --set full --clock-control none -k regex:"stats_small|score_small|scan" -s 6 -c 3 -o gpurun_out/prof_c2 python bench.py --config 2 --steps 4 --warmup 3 --no-cpu --quick > gpurun_out/ncu_c2.log 2>&1; echo "ncu c2 exit $?"
for r in srp c1 c2; do python tools/ncu_summary.py gpurun_out/prof_$r.ncu-rep > gpurun_out/ncu_${r}_summary.txt 2>&1; done
timeout 300 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu --quick > gpurun_out/bench_c2.log 2>&1; echo "c2 exit $?"
timeout 300 python bench.py --config 3 --mode srp --steps 10 --warmup 3 --no-cpu --quick > gpurun_out/bench_c3srp.log 2>&1; echo "c3 srp exit $?"
for n in 2 4 8; do timeout 300 python bench.py --shard-of $n --no-cpu --quick > gpurun_out/shard_$n.log 2>&1; done; echo "shards done"

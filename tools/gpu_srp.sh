# SRP (d = 5, the reference default) on configs[3] / [2] / [1]: kernel split + ncu of stats_small
cd $GRAFT_REPO_ROOT
for c in 3 2; do
timeout 300 python bench.py --config $c --mode srp --steps 10 --warmup 3 --no-cpu --quick > gpurun_out/srp_c$c.log 2>&1; echo "c$c exit $?"; python tools/bench_summary.py gpurun_out/srp_c$c.log 2>/dev/null | head -7
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"stats_small|score_small" -s 4 -c 2 -o gpurun_out/prof_srp python bench.py --config 3 --mode srp --steps 4 --warmup 3 --no-cpu --quick > gpurun_out/ncu_srp.log 2>&1; echo "ncu exit $?"
python tools/ncu_summary.py gpurun_out/prof_srp.ncu-rep

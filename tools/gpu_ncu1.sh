# one ncu --set full capture of kernel regex $NCU_K on the c3 bench (source-correlated)
cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$NCU_K" -s 2 -c 1 -o gpurun_out/prof_1 python bench.py --steps 4 --warmup 3 --no-cpu --quick ${BENCH_ARGS} > gpurun_out/ncu_1.log 2>&1; echo "ncu exit $?"
python tools/ncu_summary.py gpurun_out/prof_1.ncu-rep | head -30

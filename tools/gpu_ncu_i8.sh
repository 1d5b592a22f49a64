# ncu full capture of the exact-int8 stats kernel
set -x
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "stats" > gpurun_out/pytest_i8.log 2>&1; echo "pytest exit $?"
tail -3 gpurun_out/pytest_i8.log
timeout 300 python bench.py --steps 4 --warmup 3 --no-cpu --quick --stats 2 > gpurun_out/plain_i8.log 2>&1; echo "plain exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stats_i8" -s 2 -c 1 -o gpurun_out/prof_st8 python bench.py --steps 4 --warmup 3 --no-cpu --quick --stats 2 > gpurun_out/ncu_i8.log 2>&1; echo "ncu exit $?"

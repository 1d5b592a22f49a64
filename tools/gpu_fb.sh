cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "factor or determin or config4 or c4" > gpurun_out/pytest_fb.log 2>&1; echo "pytest exit $?"
tail -3 gpurun_out/pytest_fb.log
for w in 32 1; do timeout 300 python bench.py --config 4 --window $w --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_c4_$w.log 2>&1; echo "bench c4 w$w exit $?"; python tools/bench_summary.py gpurun_out/bench_c4_$w.log; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"factor|stats|score|scan" -c 40 --csv python bench.py --config 4 --window 32 --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_c4.csv 2>/dev/null; echo "ncu exit $?"
grep -E "factor|stats|score|scan" gpurun_out/ncu_c4.csv | awk -F'","' '{print $5, $NF}' | sort | uniq -c | head -20

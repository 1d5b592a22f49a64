# per-config kernel breakdowns (device-resident), quick
cd $GRAFT_REPO_ROOT
for c in "1 full 16" "1 srp 64" "2 full 256" "2 srp 256" "4 full 8" "4 srp 32" "0 full 64" "3 srp 16"; do
  set -- $c
  timeout 600 python bench.py --config $1 --mode $2 --window $3 --steps 6 --warmup 2 --no-cpu --quick > gpurun_out/bench_c$1_$2.log 2>&1; echo "c$1 $2 exit $?"
done

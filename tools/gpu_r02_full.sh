# round-2 evidence run: full GPU tests (parity table), bench, reference arm, launch list
export ERX_PARITY_LOG=gpurun_out/parity_r02.jsonl
rm -f $ERX_PARITY_LOG
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --tb=short > gpurun_out/gputests_r02.log 2>&1
tail -3 gpurun_out/gputests_r02.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err; echo bench rc=$?
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref_r02.json 2>&1; echo ref rc=$?
python bench.py --steps 2 --warmup 1 --quick --no-cpu > gpurun_out/plain_launch.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_r02.csv \
    python bench.py --steps 2 --warmup 1 --quick --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?

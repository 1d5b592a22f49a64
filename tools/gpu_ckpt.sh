# checkpoint: full GPU tests + bench at the working tree
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --tb=short > gpurun_out/gputests_ckpt.log 2>&1
tail -3 gpurun_out/gputests_ckpt.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_ckpt.json 2> gpurun_out/bench_ckpt.err; echo bench rc=$?
python tools/bench_summary.py gpurun_out/bench_ckpt.json | cut -c1-400

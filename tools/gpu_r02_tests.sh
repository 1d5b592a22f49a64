# round-2 GPU checks: edge numerics, full-length parity (appends the parity table), the rest of -m gpu
export ERX_PARITY_LOG=gpurun_out/parity_r02.jsonl
rm -f $ERX_PARITY_LOG
timeout 900 python -m pytest tests/test_gpu_numerics.py -q -p no:cacheprovider --tb=short ${NUMERICS_K:+-k "$NUMERICS_K"} 2>&1 | grep -E "^E  |passed|failed|Error" | head -40
[ -n "$SKIP_FULL" ] || timeout 900 python -m pytest tests/test_gpu_fullstream.py -q -p no:cacheprovider --tb=short 2>&1 | grep -E "^E  |passed|failed" | head -20
[ -n "$SKIP_REST" ] || timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --tb=short --deselect tests/test_gpu_fullstream.py --deselect tests/test_gpu_numerics.py 2>&1 | grep -E "^E  |passed|failed" | head -30

timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_numerics.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
python tools/kt_probe.py 2 full 2048 20
python tools/kt_probe.py 2 full 4096 20

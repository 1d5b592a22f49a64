timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_numerics.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
python tools/kt_probe.py 3 srp 64 20
python tools/kt_probe.py 3 srp 32 20
python tools/kt_probe.py 1 srp 256 20
python tools/kt_probe.py 4 srp 32 20

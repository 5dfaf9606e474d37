export PYTHONPATH=$PWD
timeout -k 10 300 python -m pytest tests/test_kernels_gpu.py tests/test_parity_gpu.py -q -x -p no:cacheprovider --timeout 100 2>&1 | tail -4
timeout -k 10 120 python tools/attn_probe.py 2>&1 | tail -5

export PYTHONPATH=$PWD
timeout -k 10 300 python -m pytest tests/test_kernels_gpu.py tests/test_parity_gpu.py tests/test_ulysses_gpu.py -q -p no:cacheprovider --timeout 200 2>&1 | tail -15
timeout -k 10 120 python tools/attn_probe.py --variant 1 2>&1 | tail -6
timeout -k 10 120 python tools/engine_fusion_probe.py 2>&1 | tail -8

export PYTHONPATH=$PWD
timeout -k 10 300 python tools/host_tier_debug.py 2>&1 | grep -v "block ctx" | tail -20
timeout -k 10 600 python -m pytest tests/test_parity_gpu.py tests/test_ulysses_gpu.py tests/test_kernels_gpu.py -q -p no:cacheprovider --timeout 600 -k "host_tier or random_ops or replay or ulysses_engine or paged or kv_append" 2>&1 | tail -3

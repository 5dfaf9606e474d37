export PYTHONPATH=$PWD
timeout -k 10 900 python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider --timeout 600 -k "graph or host_tier or engine" 2>&1 | tail -4

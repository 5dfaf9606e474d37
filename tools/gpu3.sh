export PYTHONPATH=$PWD
timeout -k 10 900 python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider --timeout 300 -s 2>&1 | tail -40

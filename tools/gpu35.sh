export PYTHONPATH=$PWD
timeout -k 10 120 python tools/attn_probe.py --cross 3 2>&1 | tail -1
IFX_NO_FEW_KEYS=1 timeout -k 10 120 python tools/attn_probe.py --cross 3 2>&1 | tail -1
timeout -k 10 300 python -m pytest tests/test_kernels_gpu.py -q -p no:cacheprovider -k attention 2>&1 | tail -2

export PYTHONPATH=$PWD
timeout -k 10 300 python -m pytest tests/test_kernels_gpu.py tests/test_parity_gpu.py tests/test_ulysses_gpu.py -q -x -p no:cacheprovider --timeout 300 -k "not c3" 2>&1 | tail -3
timeout -k 10 120 python tools/attn_probe.py 2>&1 | tail -5
for h in 2 5; do echo "heads=$h split"; timeout -k 10 120 python tools/attn_probe.py --heads $h 2>&1 | tail -5; echo "heads=$h no split"; timeout -k 10 120 python tools/attn_probe.py --heads $h --no-split 2>&1 | tail -5; done

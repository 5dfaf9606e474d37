set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout -k 10 400 python -m pytest tests/test_kernels_gpu.py -q -p no:cacheprovider --timeout 120 2>&1 | tail -30
timeout -k 10 120 python tools/attn_probe.py --variant 0 2>&1 | tail -8
timeout -k 10 120 python tools/attn_probe.py --variant 1 2>&1 | tail -8

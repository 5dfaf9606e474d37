export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout -k 10 600 python -m pytest tests/test_parity_gpu.py tests/test_kernels_gpu.py -q -p no:cacheprovider --timeout 600 -k "host_tier or paged or kv_append or random_ops or replay" 2>&1 | grep -E "passed|failed|Error|assert" | head -20
timeout -k 10 120 python tools/attn_probe.py 2>&1 | tail -5; echo paged
timeout -k 10 120 python tools/attn_probe.py --paged 2>&1 | tail -5

export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout -k 10 600 python -m pytest tests/test_parity_gpu.py tests/test_kernels_gpu.py -q -p no:cacheprovider --timeout 600 -k "host_tier or paged or kv_append or random_ops" 2>&1 | tail -15
timeout -k 10 120 python tools/attn_probe.py 2>&1 | tail -5; echo paged
timeout -k 10 120 python tools/attn_probe.py --paged 2>&1 | tail -5
timeout -k 10 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 2>&1 | tail -5
timeout -k 10 900 python bench.py --no-cpu-baseline 2>&1 | tail -1 | tee gpurun_out/bench_paged.json

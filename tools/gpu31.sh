export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout -k 10 600 python -m pytest tests/test_kernels_gpu.py tests/test_parity_gpu.py -q -p no:cacheprovider --timeout 600 -k "attention or host_tier or engine_tiny or engine_small" 2>&1 | tail -3
timeout -k 10 1500 python bench.py --config c5 --steps 2 > gpurun_out/c5.log 2>&1; tail -3 gpurun_out/c5.log
timeout -k 10 900 python bench.py --no-cpu-baseline 2>&1 | tail -1 | tee gpurun_out/bench_r03_c2.json

export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout -k 10 600 python -m pytest tests/test_parity_gpu.py tests/test_ulysses_gpu.py -q -p no:cacheprovider --timeout 600 -k "host_tier or random_ops or replay or ulysses_engine" 2>&1 | tail -3
timeout -k 10 1500 python bench.py --config c5 --steps 2 2>&1 | tail -3 | tee gpurun_out/bench_r03_c5.json

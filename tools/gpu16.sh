export PYTHONPATH=$PWD
timeout -k 10 300 python -m pytest tests/test_kernels_gpu.py tests/test_parity_gpu.py -q -x -p no:cacheprovider --timeout 300 -k "not c3" 2>&1 | tail -2
timeout -k 10 120 python tools/kv_probe.py 2>&1 | tail -3
timeout -k 10 900 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | tee gpurun_out/bench_c4_r02.json

export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout -k 10 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 2>&1 | tail -4
timeout -k 10 300 python tools/host_cost_probe.py 2>&1 | tail -1
timeout -k 10 900 python bench.py --no-cpu-baseline 2>&1 | tail -1 | tee gpurun_out/bench_r03_c2.json

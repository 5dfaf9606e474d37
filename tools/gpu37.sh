export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout -k 10 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 2>&1 | tail -3
timeout -k 10 900 python bench.py 2>&1 | tail -1 | tee gpurun_out/bench_r03_c2.json
timeout -k 10 1800 python bench.py --config c5 --steps 2 > gpurun_out/c5.log 2>&1; tail -1 gpurun_out/c5.log | tee gpurun_out/bench_r03_c5.json

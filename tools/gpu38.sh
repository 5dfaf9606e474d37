export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout -k 10 900 python bench.py --config c3 --steps 1 --no-cpu-baseline 2>&1 | tail -1 | tee gpurun_out/bench_r03_c3.json
timeout -k 10 900 python bench.py --config c4 --steps 2 --no-cpu-baseline 2>&1 | tail -1 | tee gpurun_out/bench_r03_c4.json

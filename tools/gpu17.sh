export PYTHONPATH=$PWD
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout -k 10 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider --timeout 600 2>&1 | tail -5
timeout -k 10 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout -k 10 900 python bench.py 2>&1 | tail -1 | tee gpurun_out/bench_r03.json

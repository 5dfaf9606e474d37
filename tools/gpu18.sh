export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout -k 10 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider --timeout 600 2>&1 | tail -15
timeout -k 10 120 python tools/kv_probe.py 2>&1 | tail -5
timeout -k 10 120 python tools/attn_probe.py 2>&1 | tail -5; echo paged
timeout -k 10 900 python bench.py --no-cpu-baseline 2>&1 | tail -1 | tee gpurun_out/bench_paged.json
timeout -k 10 120 python tools/attn_probe.py --paged 2>&1 | tail -5

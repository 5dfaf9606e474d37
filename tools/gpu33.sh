export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout -k 10 120 python tools/attn_probe.py --cross 3 2>&1 | tail -1
IFX_NO_FEW_KEYS=1 timeout -k 10 120 python tools/attn_probe.py --cross 3 2>&1 | tail -1
timeout -k 10 1800 python bench.py --config c5 --steps 2 > gpurun_out/c5.log 2>&1; tail -1 gpurun_out/c5.log | tee gpurun_out/bench_r03_c5.json

export PYTHONPATH=$PWD
timeout -k 10 600 python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider --timeout 500 -k "c3" 2>&1 | tail -3
IFX_DIST_BACKEND=gloo timeout -k 10 300 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --config c1 --steps 2 --warmup 3 2>&1 | grep -v Warning | tail -3
timeout -k 10 900 python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | tee gpurun_out/bench_c3_r02.json

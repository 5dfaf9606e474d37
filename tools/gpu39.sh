export PYTHONPATH=$PWD
timeout -k 10 900 python -m pytest tests/test_ulysses_gpu.py -q -p no:cacheprovider --timeout 600 2>&1 | tail -15
IFX_DIST_BACKEND=gloo timeout -k 10 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 1 --warmup 3 --config c1 2>&1 | tail -2

export PYTHONPATH=$PWD
timeout 1800 python -m pytest tests/test_ulysses_gpu.py -x -q > gpurun_out/n_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/n_tests.log
IFX_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29616 bench.py --gpus 2 --config c1 --steps 2 --warmup 3 > gpurun_out/n_c1w2.json 2> gpurun_out/n_c1w2.err; echo c1w2 rc=$?; tail -c 600 gpurun_out/n_c1w2.json

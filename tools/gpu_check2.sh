export PYTHONPATH=$PWD
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/c2_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/c2_tests.log
IFX_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 2 --warmup 3 > gpurun_out/c2_w2.json 2> gpurun_out/c2_w2.err; echo w2 rc=$?; tail -c 600 gpurun_out/c2_w2.json; tail -3 gpurun_out/c2_w2.err
timeout 800 python tools/e2e_probe.py --n 4 > gpurun_out/e2e2.log 2>&1; cat gpurun_out/e2e2.log

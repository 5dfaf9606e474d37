export PYTHONPATH=$PWD
timeout 1800 python -m pytest tests/test_ulysses_gpu.py -x -q -k "p2p" > gpurun_out/g_uly.log 2>&1; echo uly rc=$?; tail -3 gpurun_out/g_uly.log
timeout 900 python tools/rank_probe.py --configs c2 --worlds 1 8 --rollouts 2 2>/dev/null
IFX_DIST_BACKEND=gloo timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29615 bench.py --gpus 2 --config c1 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/g_c1w2.json 2> gpurun_out/g_c1w2.err; echo c1w2 rc=$?; tail -c 300 gpurun_out/g_c1w2.json

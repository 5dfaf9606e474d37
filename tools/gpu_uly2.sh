export PYTHONPATH=$PWD
timeout 1800 python -m pytest tests/test_ulysses_gpu.py -x -q > gpurun_out/v_uly.log 2>&1; echo uly rc=$?; tail -3 gpurun_out/v_uly.log
IFX_DIST_BACKEND=gloo timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29613 bench.py --gpus 2 --config c4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/v_c4w2.json 2> gpurun_out/v_c4w2.err; echo c4w2 rc=$?
IFX_DIST_BACKEND=gloo timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29614 bench.py --gpus 4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/v_c2w4.json 2> gpurun_out/v_c2w4.err; echo c2w4 rc=$?
for f in v_c4w2 v_c2w4; do echo "== $f"; tail -c 700 gpurun_out/$f.json; grep -v "OMP_NUM\|\*\*\*\*" gpurun_out/$f.err | tail -5; done

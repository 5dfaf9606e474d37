# Ulysses engine on one B200: exchange overhead at N = 1 (p2p vs nccl), then the N > 1 bench
# path with ranks sharing the GPU over gloo (functional check of bench.py --gpus N; timings
# of time-sliced ranks are meaningless)
timeout 900 python bench.py --ulysses --exchange p2p --no-cpu-baseline > gpurun_out/u_p2p.json 2> gpurun_out/u_p2p.err; echo p2p rc=$?
timeout 900 python bench.py --ulysses --exchange nccl --no-cpu-baseline > gpurun_out/u_nccl.json 2> gpurun_out/u_nccl.err; echo nccl rc=$?
IFX_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 3 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 3 --config c1 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/u_c1w3.json 2> gpurun_out/u_c1w3.err; echo c1w3 rc=$?
IFX_DIST_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 2 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/u_c2w2.json 2> gpurun_out/u_c2w2.err; echo c2w2 rc=$?
for f in u_p2p u_nccl u_c1w3 u_c2w2; do echo "== $f"; tail -c 1200 gpurun_out/$f.json; tail -5 gpurun_out/$f.err; done

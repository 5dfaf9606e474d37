export PYTHONPATH=$PWD
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout -k 10 600 python bench.py 2>&1 | tail -3 | tee gpurun_out/bench_r01.json
timeout -k 10 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1; echo ncu1 rc=$?
timeout -k 10 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 2 -c 1 -o gpurun_out/attn_b3 python tools/ncu_attn.py 3 > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
ls -la gpurun_out

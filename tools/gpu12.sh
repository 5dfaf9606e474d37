export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout -k 10 1200 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/block6/" --csv --log-file gpurun_out/launches_r02_block6.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_r02.log 2>&1; echo ncu1 rc=$?
timeout -k 10 400 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 2 -c 1 -o gpurun_out/attn_v5_b3 python tools/ncu_attn.py 3 > gpurun_out/ncu_full_r02.log 2>&1; echo ncu2 rc=$?
timeout -k 10 400 ncu --set full --clock-control none -k regex:append -s 2 -c 1 -o gpurun_out/append_c2 python tools/ncu_append.py > gpurun_out/ncu_append.log 2>&1; echo ncu3 rc=$?

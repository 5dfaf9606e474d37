export PYTHONPATH=$PWD
mkdir -p gpurun_out
grep MemAvailable /proc/meminfo
timeout -k 10 1500 python bench.py --config c5 --steps 2 2>&1 | tail -2 | tee gpurun_out/bench_r03_c5.json
timeout -k 10 300 ncu --set full --clock-control none -k regex:append -s 2 -c 1 -o gpurun_out/append_r03 python tools/ncu_append.py > gpurun_out/ncu_append.log 2>&1; echo ncu_append rc=$?
timeout -k 10 1200 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/block6/" --csv --log-file gpurun_out/launches_r03_block6.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_r03.log 2>&1; echo ncu_launch rc=$?

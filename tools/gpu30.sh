export PYTHONPATH=$PWD
mkdir -p gpurun_out
grep -E "MemAvailable|MemTotal|Hugepages|Mlocked|Unevictable" /proc/meminfo; ulimit -l
timeout -k 10 1500 python bench.py --config c5 --steps 2 > gpurun_out/c5.log 2>&1; tail -30 gpurun_out/c5.log
timeout -k 10 300 python tools/fa4_probe.py 2>&1 | tail -6

export PYTHONPATH=$PWD
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/l_tests.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/l_tests.log
timeout 800 python tools/gap_probe.py > gpurun_out/gap4.log 2>&1; grep "GPU span" gpurun_out/gap4.log; sed -n 2,6p gpurun_out/gap4.log; rm -f gpurun_out/gap_trace.json
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],3), d['e2e']['ms_each'], round(d['e2e']['value'],3), d['clocks']['sm_mhz'])"; done

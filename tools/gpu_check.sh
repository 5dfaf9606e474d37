export PYTHONPATH=$PWD
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/c_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/c_tests.log
timeout 800 python tools/gap_probe.py > gpurun_out/gap2.log 2>&1; head -12 gpurun_out/gap2.log
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline > gpurun_out/c_b$i.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/c_b$i.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['achieved'], d['host_enqueue_ms_per_step'], d['clocks']['sm_mhz'])"; done

export PYTHONPATH=$PWD
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/f_smoke.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/f_tests.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/f_tests.log
timeout 900 python bench.py > gpurun_out/f_c2.json 2> gpurun_out/f_c2.err; echo c2 rc=$?
python -c "import json; d=json.loads(open('gpurun_out/f_c2.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e'], d['roofline']['achieved'], d['clocks'], d['cpu_baseline']['value'])"

export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_ulysses_gpu.py -x -q -k "graph or c2 or ulysses" > gpurun_out/v_tests.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/v_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/v_c2.json 2>gpurun_out/v_err.log; echo bench rc=$?
python -c "import json; d=json.loads(open('gpurun_out/v_c2.json').read().strip().splitlines()[-1]); print(round(d['value'],3), d['e2e'], round(d['roofline']['achieved'],1), d['roofline']['launches'], round(d['roofline']['share_of_step'],3), d['gpu_launches'], d['clocks'])"

export PYTHONPATH=$PWD
timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_ulysses_gpu.py -x -q -k "graph or ulysses_engine or nccl" > gpurun_out/h2_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/h2_tests.log
timeout 900 python tools/rank_probe.py --configs c2 --worlds 1 8 --rollouts 2 --profile 2>/dev/null | grep -v top_gaps | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l)
    if 'profile' in d: print('profile', d['world'], d['span_ms'], d['kernel_ms'], d['gap_ms_by_size'])
    else: print(d['world'], d['ms_rank'], d['k1_ms'], d['strong_scaling_bound'])"
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/h2_c2.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/h2_c2.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'])"

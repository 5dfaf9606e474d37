export PYTHONPATH=$PWD
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/f_smoke.log
timeout 2700 python -m pytest tests -m gpu -q > gpurun_out/f_gpu.log 2>&1; echo gputests rc=$?; tail -2 gpurun_out/f_gpu.log
timeout 900 python bench.py > gpurun_out/f_c2.json 2> gpurun_out/f_c2.err; echo c2 rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/f_ref.json 2> gpurun_out/f_ref.err; echo ref rc=$?
timeout 1200 python tools/rank_probe.py --configs c2 c4 --worlds 1 2 4 8 --rollouts 2 2>/dev/null | grep "^{" > gpurun_out/f_rank.jsonl; echo rank rc=$?
for f in f_c2 f_ref; do python -c "import json; d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]); print('$f', d['value'], d['e2e']['value'], d.get('roofline',{}).get('frac'))"; done
cat gpurun_out/f_rank.jsonl | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['config'], d['world'], d['ms_rank'], d['strong_scaling_bound'], d['head_split'], d['g1_fused_norms'])"

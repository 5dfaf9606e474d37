export PYTHONPATH=$PWD
for i in 1 2; do for v in 1 0; do
  IFX_HOST_BOUND_CAPTURE=$v timeout 600 python bench.py --no-cpu-baseline > gpurun_out/hb_${v}_$i.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/hb_${v}_$i.json').read().strip().splitlines()[-1]); print('bench hb=$v', d['value'], d['e2e']['value'])"
done; done
for v in 1 0; do echo "== hb $v"; IFX_HOST_BOUND_CAPTURE=$v timeout 900 python tools/rank_probe.py --configs c2 c4 --worlds 1 8 --rollouts 2 2>/dev/null | grep "^{"; done

export PYTHONPATH=$PWD
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/k_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/k_tests.log
IFX_K1_GRID=items timeout 300 python tools/attn_probe.py --paged > gpurun_out/k_items.log 2>&1; echo items; cat gpurun_out/k_items.log
timeout 300 python tools/attn_probe.py --paged > gpurun_out/k_pers.log 2>&1; echo persistent; cat gpurun_out/k_pers.log
for i in 1 2; do
  IFX_K1_GRID=items timeout 600 python bench.py --no-cpu-baseline > gpurun_out/kb_items_$i.json 2>/dev/null
  timeout 600 python bench.py --no-cpu-baseline > gpurun_out/kb_pers_$i.json 2>/dev/null
done
for f in gpurun_out/kb_*.json; do echo $f; python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['achieved'], d['clocks']['sm_mhz'])"; done

#!/bin/bash
# K1 A/B on the final build: exp2 pairs (of every 8) on the FMA pipe, 0 / 1 / 2 (default) / 3.
export PYTHONPATH=$PWD
for v in base poly0 poly1 poly3; do
  if [ $v = base ]; then unset IFX_LIB_PATH; else export IFX_LIB_PATH=$PWD/build_ab_$v.so; fi
  echo "== probe $v"; timeout 300 python tools/attn_probe.py --paged 2>&1 | grep '^{'
done
for i in 1 2; do
  for v in base poly0 poly1 poly3; do
    if [ $v = base ]; then unset IFX_LIB_PATH; else export IFX_LIB_PATH=$PWD/build_ab_$v.so; fi
    timeout 600 python bench.py --no-cpu-baseline > gpurun_out/pp_${v}_$i.json 2>/dev/null
  done
done
unset IFX_LIB_PATH
for f in gpurun_out/pp_*.json; do echo $f; python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['achieved'], d['clocks']['sm_mhz'])"; done

#!/bin/bash
# K1 A/B: key half 1 started out of phase with half 0 at each item (IFX_K1_STAGGER cycles).
export PYTHONPATH=$PWD
for v in base st300 st700 st1200; do
  if [ $v = base ]; then unset IFX_LIB_PATH; else export IFX_LIB_PATH=$PWD/build_ab_$v.so; fi
  echo "== probe $v"; timeout 300 python tools/attn_probe.py --paged 2>&1 | grep '^{'
done
for i in 1 2; do
  for v in base st300 st700 st1200; do
    if [ $v = base ]; then unset IFX_LIB_PATH; else export IFX_LIB_PATH=$PWD/build_ab_$v.so; fi
    timeout 600 python bench.py --no-cpu-baseline > gpurun_out/st_${v}_$i.json 2>/dev/null
  done
done
unset IFX_LIB_PATH
for f in gpurun_out/st_*.json; do echo $f; python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['achieved'], d['clocks']['sm_mhz'])"; done

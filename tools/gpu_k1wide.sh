#!/bin/bash
# K1 A/B: S read by one tcgen05.ld 32x32b.x64 and P written by one .x32 store (IFX_K1_WIDE=1)
# vs two x32 loads / two x16 stores.
export PYTHONPATH=$PWD
IFX_LIB_PATH=$PWD/build_ab_wide.so timeout 900 python -m pytest tests/test_kernels_gpu.py -x -q 2>&1 | tail -2
for v in base wide; do
  if [ $v = base ]; then unset IFX_LIB_PATH; else export IFX_LIB_PATH=$PWD/build_ab_$v.so; fi
  echo "== probe $v"; timeout 300 python tools/attn_probe.py --paged 2>&1 | grep '^{'
done
for i in 1 2; do
  for v in base wide; do
    if [ $v = base ]; then unset IFX_LIB_PATH; else export IFX_LIB_PATH=$PWD/build_ab_$v.so; fi
    timeout 600 python bench.py --no-cpu-baseline > gpurun_out/kw_${v}_$i.json 2>/dev/null
  done
done
unset IFX_LIB_PATH
for f in gpurun_out/kw_*.json; do echo $f; python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['achieved'], d['clocks']['sm_mhz'])"; done

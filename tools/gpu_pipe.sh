export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_kernels_gpu.py -x -q > gpurun_out/pp_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/pp_tests.log
for v in pipe nopipe; do
  if [ $v = nopipe ]; then export IFX_LIB_PATH=$PWD/build_ab_nopipe.so; else unset IFX_LIB_PATH; fi
  echo "probe $v"; timeout 300 python tools/attn_probe.py --paged 2>/dev/null | tail -5
  echo "probe5 $v"; timeout 300 python tools/attn_probe.py --paged --heads 5 2>/dev/null | tail -5
done
for i in 1 2; do
  for v in pipe nopipe; do
    if [ $v = nopipe ]; then export IFX_LIB_PATH=$PWD/build_ab_nopipe.so; else unset IFX_LIB_PATH; fi
    timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ppb_${v}_$i.json 2>/dev/null
    python -c "import json; d=json.loads(open('gpurun_out/ppb_${v}_$i.json').read().strip().splitlines()[-1]); print('$v', d['value'], d['e2e']['value'], d['roofline']['achieved'], d['clocks']['sm_mhz'])"
  done
done

export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_kernels_gpu.py -x -q > gpurun_out/q_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/q_tests.log
for v in quarters halves; do
  if [ $v = halves ]; then export IFX_LIB_PATH=$PWD/build_ab_halves.so; else unset IFX_LIB_PATH; fi
  timeout 300 python tools/attn_probe.py --paged > gpurun_out/q_probe_$v.log 2>&1; echo probe $v; tail -5 gpurun_out/q_probe_$v.log
  timeout 300 python tools/attn_probe.py --paged --heads 5 > gpurun_out/q_probe5_$v.log 2>&1; echo probe5 $v; tail -5 gpurun_out/q_probe5_$v.log
done
for i in 1 2; do
  for v in quarters halves; do
    if [ $v = halves ]; then export IFX_LIB_PATH=$PWD/build_ab_halves.so; else unset IFX_LIB_PATH; fi
    timeout 600 python bench.py --no-cpu-baseline > gpurun_out/qb_${v}_$i.json 2>/dev/null
  done
done
unset IFX_LIB_PATH
for f in gpurun_out/qb_*.json; do echo $f; python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['achieved'], d['clocks']['sm_mhz'])"; done

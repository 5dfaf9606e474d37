export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_seqpar_gpu.py tests/test_acceptance_gpu.py -x -q > gpurun_out/p_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/p_tests.log
for v in parity halves; do
  if [ $v = halves ]; then export IFX_LIB_PATH=$PWD/build_ab_halves.so; else unset IFX_LIB_PATH; fi
  timeout 300 python tools/attn_probe.py --paged > gpurun_out/p_probe_$v.log 2>&1; echo probe $v; tail -6 gpurun_out/p_probe_$v.log
  timeout 300 python tools/attn_probe.py --paged --heads 5 > gpurun_out/p_probe5_$v.log 2>&1; echo probe5 $v; tail -6 gpurun_out/p_probe5_$v.log
done
for i in 1 2; do
  for v in parity halves; do
    if [ $v = halves ]; then export IFX_LIB_PATH=$PWD/build_ab_halves.so; else unset IFX_LIB_PATH; fi
    timeout 600 python bench.py --no-cpu-baseline > gpurun_out/pb_${v}_$i.json 2>/dev/null
  done
done
unset IFX_LIB_PATH
for f in gpurun_out/pb_*.json; do echo $f; python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['achieved'], d['clocks']['sm_mhz'])"; done

export PYTHONPATH=$PWD
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/d_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/d_tests.log
for i in 1 2; do
  for v in 1 0; do
    IFX_PDL=$v timeout 600 python bench.py --no-cpu-baseline > gpurun_out/db_${v}_$i.json 2>/dev/null
  done
done
for f in gpurun_out/db_*.json; do echo $f; python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['achieved'], d['clocks']['sm_mhz'])"; done
for v in 1 0; do echo "== PDL $v"; IFX_PDL=$v timeout 900 python tools/rank_probe.py --configs c2 c4 --worlds 8 --rollouts 2 2>/dev/null; done

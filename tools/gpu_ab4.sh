export PYTHONPATH=$PWD
for i in 1 2 3; do for v in base lt16; do
  IFX_LIB_PATH=$PWD/build_ab_$v.so timeout 600 python bench.py --no-cpu-baseline > gpurun_out/g_${v}_$i.json 2>/dev/null
  echo "$v run $i: $(python -c "import json; d=json.loads(open('gpurun_out/g_${v}_$i.json').read().strip().splitlines()[-1]); print(round(d['value'],3), round(d['e2e']['value'],3), round(d['roofline']['achieved'],1), round(d['ms_per_step']-d['roofline']['kernel_ms_per_step'],1), d['clocks']['sm_mhz'])")"
done; done

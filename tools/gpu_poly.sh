export PYTHONPATH=$PWD
for i in 1 2 3; do for v in 0 1 2; do
  IFX_LIB_PATH=$PWD/build_ab_poly$v.so timeout 600 python bench.py --no-cpu-baseline > gpurun_out/p_${v}_$i.json 2>/dev/null
  echo "poly $v run $i: $(python -c "import json; d=json.loads(open('gpurun_out/p_${v}_$i.json').read().strip().splitlines()[-1]); print(round(d['value'],3), round(d['e2e']['value'],3), round(d['roofline']['achieved'],1), d['clocks']['sm_mhz'], d['clocks']['power_w_max'])")"
done; done
for v in 0 1; do echo "probe poly $v"; IFX_LIB_PATH=$PWD/build_ab_poly$v.so python tools/attn_probe.py --paged; done

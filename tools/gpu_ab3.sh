export PYTHONPATH=$PWD
IFX_LIB_PATH=$PWD/build_ab_unroll.so timeout 300 python -m pytest tests/test_kernels_gpu.py -q -x -k "attention" 2>&1 | tail -1
for v in base unroll base unroll; do echo "probe $v"; IFX_LIB_PATH=$PWD/build_ab_$v.so python tools/attn_probe.py --paged; done
for i in 1 2; do for v in base unroll; do
  IFX_LIB_PATH=$PWD/build_ab_$v.so timeout 600 python bench.py --no-cpu-baseline > gpurun_out/u_${v}_$i.json 2>/dev/null
  echo "$v run $i: $(python -c "import json; d=json.loads(open('gpurun_out/u_${v}_$i.json').read().strip().splitlines()[-1]); print(round(d['value'],3), round(d['e2e']['value'],3), round(d['roofline']['achieved'],1), d['clocks']['sm_mhz'])")"
done; done

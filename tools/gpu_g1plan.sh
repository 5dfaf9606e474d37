export PYTHONPATH=$PWD
for cfg in "0 0" "3 256" "3 128" "1 256" "1 192" "1 128"; do
  set -- $cfg
  echo "== mode $1 bn $2"
  if [ $1 = 0 ]; then unset IFX_G1_MODE IFX_G1_BN; else export IFX_G1_MODE=$1 IFX_G1_BN=$2; fi
  timeout 300 python tools/scatter_probe.py 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['cfg'], d['world'], d['M'], 'lt', d['cublaslt_us'], 'g1', d['g1_us'], 'sc', d['g1_scatter_us'])"
done

export PYTHONPATH=$PWD
for v in 1 11 12 13 0; do echo "variant $v"; timeout -k 10 60 python tools/attn_probe.py --variant $v --quick 2>&1 | tail -1; done

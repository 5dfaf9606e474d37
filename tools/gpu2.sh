export PYTHONPATH=$PWD
timeout -k 10 120 python tools/attn_probe.py --variant 0 2>&1 | tail -8
timeout -k 10 120 python tools/attn_probe.py --variant 1 2>&1 | tail -8

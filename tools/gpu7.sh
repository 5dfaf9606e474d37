export PYTHONPATH=$PWD
timeout -k 10 300 python -m pytest tests/test_kernels_gpu.py -q -x -p no:cacheprovider --timeout 100 -k attention 2>&1 | tail -15
for v in 4 5 3; do echo "variant $v"; timeout -k 10 120 python tools/attn_probe.py --variant $v 2>&1 | tail -5; done

export PYTHONPATH=$PWD
cp tools/lib_nowait.so paper_2511_20714_b200/libinferix_b200.so
timeout -k 10 300 python -m pytest tests/test_kernels_gpu.py tests/test_parity_gpu.py -q -x -p no:cacheprovider --timeout 100 2>&1 | tail -3
timeout -k 10 120 python tools/attn_probe.py 2>&1 | tail -5

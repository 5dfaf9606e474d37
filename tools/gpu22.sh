export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout -k 10 600 python -m pytest tests/test_parity_gpu.py tests/test_kernels_gpu.py -q -p no:cacheprovider --timeout 600 -k "host_tier or paged or attention" 2>&1 | tail -3
timeout -k 10 120 python tools/attn_probe.py 2>&1 | tail -5; echo paged
timeout -k 10 120 python tools/attn_probe.py --paged 2>&1 | tail -5
timeout -k 10 400 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 2 -c 1 -o gpurun_out/attn_paged2_b6 python tools/ncu_attn.py 6 --paged > gpurun_out/ncu_p.log 2>&1; echo ncu2 rc=$?

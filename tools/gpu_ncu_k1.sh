export PYTHONPATH=$PWD
timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -k "persistent or attention" > gpurun_out/n_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/n_tests.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 2 -c 1 -o gpurun_out/attn_pers_b6 -f python tools/ncu_attn.py 6 --paged > gpurun_out/n_b6.log 2>&1; echo ncu6 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 2 -c 1 -o gpurun_out/attn_pers_b0 -f python tools/ncu_attn.py 0 --paged > gpurun_out/n_b0.log 2>&1; echo ncu0 rc=$?

timeout 900 python -m pytest tests/test_seqpar_gpu.py -x -q > gpurun_out/s_seqpar.log 2>&1; echo seqpar rc=$?
timeout 600 python -m pytest tests/test_peer_gpu.py tests/test_kernels_gpu.py -x -q > gpurun_out/s_kern.log 2>&1; echo kern rc=$?
tail -40 gpurun_out/s_seqpar.log; tail -5 gpurun_out/s_kern.log

export PYTHONPATH=$PWD
timeout 1500 python -m pytest tests/test_kernels_gpu.py tests/test_parity_gpu.py tests/test_seqpar_gpu.py tests/test_peer_gpu.py -x -q > gpurun_out/f_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/f_tests.log
for v in 1 0; do echo "== fixup $v"; IFX_K1_FIXUP=$v timeout 900 python tools/rank_probe.py --configs c2 c4 --worlds 4 8 --rollouts 2 2>/dev/null; done
for v in 1 0; do echo "== probe5 fixup $v"; IFX_K1_FIXUP=$v timeout 300 python tools/attn_probe.py --paged --heads 5 2>/dev/null | tail -5; done

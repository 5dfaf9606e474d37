export PYTHONPATH=$PWD
timeout 1800 python -m pytest tests/test_ulysses_gpu.py -x -q -k "p2p" > gpurun_out/u_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/u_tests.log
timeout 1200 python tools/rank_probe.py --configs c2 c4 --worlds 1 4 8 --rollouts 2 2>/dev/null | grep "^{"

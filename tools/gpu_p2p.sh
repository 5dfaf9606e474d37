# peer-memory exchange: kernel-level tests, then the multi-process Ulysses tests
timeout 600 python -m pytest tests/test_peer_gpu.py -x -q > gpurun_out/p_peer.log 2>&1; echo peer rc=$?
timeout 1500 python -m pytest tests/test_ulysses_gpu.py -x -q -k "p2p" > gpurun_out/p_uly.log 2>&1; echo uly rc=$?
tail -30 gpurun_out/p_peer.log; tail -40 gpurun_out/p_uly.log

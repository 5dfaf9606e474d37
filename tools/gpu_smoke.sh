python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/s_smoke.log 2>&1; echo smoke rc=$?
tail -3 gpurun_out/s_smoke.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/s_tests.log

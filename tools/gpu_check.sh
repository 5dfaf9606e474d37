# One GPU call: GPU tests, smoke, c2 bench (HEAD health check)
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/k_smoke.log 2>&1; echo smoke rc=$?
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/k_gputest.log 2>&1; echo gputest rc=$?
timeout 900 python bench.py > gpurun_out/k_c2.json 2> gpurun_out/k_c2.err; echo c2 rc=$?
tail -3 gpurun_out/k_gputest.log; tail -c 600 gpurun_out/k_c2.json

python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r_smoke.log 2>&1; echo smoke rc=$?
timeout 900 python bench.py > gpurun_out/r_c2.json 2> gpurun_out/r_c2.err; echo c2 rc=$?
timeout 900 python bench.py --config c3 --no-cpu-baseline > gpurun_out/r_c3.json 2> gpurun_out/r_c3.err; echo c3 rc=$?
timeout 900 python bench.py --config c4 --no-cpu-baseline > gpurun_out/r_c4.json 2> gpurun_out/r_c4.err; echo c4 rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r_ref.json 2> gpurun_out/r_ref.err; echo ref rc=$?
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/block6/" --csv --log-file gpurun_out/r_launch.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r_launch.log 2>&1; echo ncu rc=$?
tail -c 1500 gpurun_out/r_c2.json gpurun_out/r_c3.json gpurun_out/r_c4.json gpurun_out/r_ref.json

export PYTHONPATH=$PWD
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r5_smoke.log 2>&1; echo smoke rc=$?
timeout 900 python bench.py > gpurun_out/r5_c2.json 2> gpurun_out/r5_c2.err; echo c2 rc=$?
timeout 900 python bench.py --rope --no-cpu-baseline > gpurun_out/r5_c2rope.json 2> gpurun_out/r5_c2rope.err; echo c2rope rc=$?
timeout 900 python bench.py --config c3 --no-cpu-baseline > gpurun_out/r5_c3.json 2> gpurun_out/r5_c3.err; echo c3 rc=$?
timeout 900 python bench.py --config c4 --no-cpu-baseline > gpurun_out/r5_c4.json 2> gpurun_out/r5_c4.err; echo c4 rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r5_ref.json 2> gpurun_out/r5_ref.err; echo ref rc=$?
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/block6/" --csv --log-file gpurun_out/r5_launch.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r5_launch.log 2>&1; echo ncu rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 2 -c 1 -o gpurun_out/r5_k1_b6 -f python tools/ncu_attn.py 6 --paged > gpurun_out/r5_ncu_k1.log 2>&1; echo ncuk1 rc=$?
for f in r5_c2 r5_c2rope r5_c3 r5_c4 r5_ref; do echo "== $f"; tail -c 400 gpurun_out/$f.json; done

export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout -k 10 300 ncu --set full --clock-control none --import-source on -k regex:attn_fwd_v3 -s 2 -c 1 -o gpurun_out/attn_v3_b3 python tools/ncu_attn.py 3 3 > gpurun_out/ncu_v3.log 2>&1; echo rc=$?

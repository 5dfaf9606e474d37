#!/bin/bash
# ncu --set full of K1 (final build) at the c2 shape, b = 6 cached blocks.
export PYTHONPATH=$PWD
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 2 -c 1 -o gpurun_out/r5f_k1_b6 -f python tools/ncu_attn.py 6 --paged > gpurun_out/r5f_ncu_k1.log 2>&1; echo ncuk1 rc=$?
ncu -i gpurun_out/r5f_k1_b6.ncu-rep --page raw --csv > gpurun_out/r5f_k1_raw.csv 2>/dev/null; echo raw rc=$?

export PYTHONPATH=$PWD
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 2 -c 1 -o gpurun_out/k1_b6 -f python tools/ncu_attn.py 6 --paged > gpurun_out/n_b6.log 2>&1; echo ncu6 rc=$?
ncu -i gpurun_out/k1_b6.ncu-rep --page source --csv --print-source sass > gpurun_out/k1_b6_sass.csv 2>&1; echo src rc=$?
ncu -i gpurun_out/k1_b6.ncu-rep --page raw --csv > gpurun_out/k1_b6_raw.csv 2>&1
ls -la gpurun_out/k1_b6*

export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout -k 10 400 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 2 -c 1 -o gpurun_out/attn_contig_b6 python tools/ncu_attn.py 6 > gpurun_out/ncu_c.log 2>&1; echo ncu1 rc=$?
timeout -k 10 400 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 2 -c 1 -o gpurun_out/attn_paged_b6 python tools/ncu_attn.py 6 --paged > gpurun_out/ncu_p.log 2>&1; echo ncu2 rc=$?
timeout -k 10 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 2>&1 | tail -3
timeout -k 10 900 python bench.py --no-cpu-baseline 2>&1 | tail -1 | tee gpurun_out/bench_paged.json

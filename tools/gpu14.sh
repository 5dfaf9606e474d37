export PYTHONPATH=$PWD
for n in 2 3 4; do cp tools/lib_poly$n.so paper_2511_20714_b200/libinferix_b200.so; echo "poly $n/8"; timeout -k 10 120 python tools/attn_probe.py 2>&1 | tail -5; done

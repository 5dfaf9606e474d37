export PYTHONPATH=$PWD
run() {  # tag b heads rows
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:attn_fwd -s 2 -c 1 --csv python tools/ncu_attn.py $2 --paged --heads $3 --rows $4 > gpurun_out/t_$1.csv 2>/dev/null
  echo "== $1 b=$2 heads=$3 rows=$4"; grep -E "dram__bytes|gpu__time" gpurun_out/t_$1.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
}
run c2w2 6 6 4680
run c2w4 6 3 4680
run c2w8 6 3 2340
run c4 2 40 4680
run c4w2 2 20 4680
run c4w4 2 10 4680
run c4w8 2 5 4680

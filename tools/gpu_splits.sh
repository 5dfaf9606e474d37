export PYTHONPATH=$PWD
for m in 16 8 4; do
  echo "== min split tiles $m"
  IFX_K1_MIN_SPLIT_TILES=$m timeout 900 python tools/rank_probe.py --configs c2 c4 --worlds 1 4 8 --rollouts 1 2>/dev/null
done

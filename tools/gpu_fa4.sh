export PYTHONPATH=$PWD
for shape in "12 4680" "5 4680" "3 2340"; do set -- $shape
  echo "== heads $1 rows $2"
  timeout 300 python tools/fa4_probe.py --heads $1 --rows $2 2>/dev/null | grep "^{"
  timeout 300 python tools/attn_probe.py --paged --heads $1 --rows $2 2>/dev/null | grep "^{"
done

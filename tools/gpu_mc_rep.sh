# MC (sin, cos) table replication A/B: default build (1 copy) vs 2/4/8 copies
for rep in 1 2; do
for v in default mcrep2 mcrep4 mcrep8; do
  if [ $v = default ]; then unset DIVUQ_LIB_PATH; else export DIVUQ_LIB_PATH=tools/variants/$v.so; fi
  python bench.py --config 2 --steps 20 --no-e2e --no-cpu 2>/dev/null | python3 -c "import json,sys;d=json.loads(sys.stdin.read());print('$v', round(d['ms_per_step'],4),'ms')"
done; done
unset DIVUQ_LIB_PATH

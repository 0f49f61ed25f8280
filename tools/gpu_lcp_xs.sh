timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -2
for rep in 1 2; do for v in default noxs; do
  if [ $v = default ]; then unset DIVUQ_LIB_PATH; else export DIVUQ_LIB_PATH=tools/variants/$v.so; fi
  for w in lcp lcpfused; do
    python bench.py --workload $w --steps 50 --no-e2e --no-cpu 2>/dev/null | python3 -c "import json,sys;d=json.loads(sys.stdin.read());print('$v $w', round(d['ms_per_step']*1e3,1),'us')"
  done; done; done

# A/B of the LCP tail evaluation: table erfc (default build) vs the fitted
# erfc + exp (tools/variants/lcpfit.so, -DDIVUQ_LCP_ERFC_TAB=0); LCP tests on the default
set -x
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "lcp or cli or reference_boundary or cell" 2>&1 | tail -3
timeout 600 python -m pytest tests/test_cli.py tests/test_lcp.py -q -p no:cacheprovider 2>&1 | tail -2
for rep in 1 2; do
for v in default fit; do
  if [ $v = fit ]; then export DIVUQ_LIB_PATH=tools/variants/lcpfit.so; else unset DIVUQ_LIB_PATH; fi
  for w in lcp lcpfused; do
    python bench.py --workload $w --steps 50 --no-e2e --no-cpu 2>/dev/null | python3 -c "import json,sys;d=json.loads(sys.stdin.read());print('$v $w', round(d['ms_per_step']*1e3,1),'us', round(d['roofline']['frac'],3))"
  done
done
done
unset DIVUQ_LIB_PATH

# LCP / fused LCP tile heights with the row-run epilogue (variants from tools/build_variant.py)
for rep in 1 2; do
for v in default lt32 lf24 lf32; do
  if [ $v = default ]; then unset DIVUQ_LIB_PATH; else export DIVUQ_LIB_PATH=tools/variants/$v.so; fi
  for w in lcp lcpfused; do
    python bench.py --workload $w --steps 50 --no-e2e --no-cpu 2>/dev/null | python3 -c "import json,sys;d=json.loads(sys.stdin.read());print('$v $w', round(d['ms_per_step']*1e3,1),'us')"
  done
done; done

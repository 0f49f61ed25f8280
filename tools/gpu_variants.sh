# A/B timing of variant libraries (tools/build_variant.py) on one bench line.
# usage: bash tools/gpu_variants.sh "<bench args>" "<pytest -k expr or ''>" lib1 lib2 ...
O=gpurun_out/variants
mkdir -p $O
args=$1; shift; kexpr=$1; shift
for rep in 1 2; do
for lib in "" "$@"; do
  n=$(basename "${lib:-default}" .so)
  if [ $rep = 1 ] && [ -n "$kexpr" ]; then
    DIVUQ_LIB_PATH=$lib timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "$kexpr" > $O/test_$n.txt 2>&1
    echo "$n tests: $(tail -1 $O/test_$n.txt)"
  fi
  DIVUQ_LIB_PATH=$lib timeout 600 python bench.py $args --no-cpu --no-fp64 > $O/b_$n.json 2> $O/b_$n.err
  python -c "import json,sys;d=json.load(open('$O/b_$n.json'));print('$n', d['ms_per_step'], d['roofline']['frac'], d.get('clocks',{}).get('sm_mhz'))" || tail -3 $O/b_$n.err
done
done

# Full-state check of HEAD on one B200: GPU tests, smoke, every bench line.
set -x
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,memory.total --format=csv > gpurun_out/box.txt
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -15
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE_OK')" 2>&1 | tail -1
for c in 3 4 1 0 2; do
  extra=""; [ $c = 4 ] && extra="--steps 20"; [ $c = 2 ] && extra="--steps 5"
  timeout 600 python bench.py --config $c $extra > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err || tail -5 gpurun_out/bench_c$c.err
done
for w in lcp gradient fit ingest redsea; do
  timeout 600 python bench.py --workload $w --steps 20 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err || tail -5 gpurun_out/bench_$w.err
done
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2>&1
for f in gpurun_out/bench_*.json; do python3 -c "
import json,sys;d=json.load(open('$f'));print('$f',round(d['ms_per_step'],4),'%.4g'%d['value'],(d.get('roofline') or {}).get('frac'),(d.get('e2e') or {}).get('value'),(d.get('cpu_baseline') or {}).get('value'))"; done

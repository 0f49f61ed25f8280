set -x
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE_OK')" 2>&1 | tail -1
for c in 3 4 1 0 2; do
  extra=""; [ $c = 4 ] && extra="--no-e2e --steps 20"; [ $c = 2 ] && extra="--steps 5"
  python bench.py --config $c $extra > gpurun_out/bench_r01_c$c.json 2> gpurun_out/bench_r01_c$c.err || tail -5 gpurun_out/bench_r01_c$c.err
done
for w in lcp gradient ingest; do
  python bench.py --workload $w --steps 20 > gpurun_out/bench_r01_$w.json 2> gpurun_out/bench_r01_$w.err || tail -5 gpurun_out/bench_r01_$w.err
done
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_r01_ref.json 2>&1
for f in gpurun_out/bench_r01_*.json; do python3 -c "
import json,sys;d=json.load(open('$f'));print('$f',round(d['ms_per_step'],4),'%.4g'%d['value'],(d.get('roofline') or {}).get('frac'),(d.get('e2e') or {}).get('value'),(d.get('cpu_baseline') or {}).get('value'))"; done
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
bash tools/gpu_prof.sh lcp lcp2d --workload lcp --steps 3 --no-cpu
bash tools/gpu_prof.sh gradient gradient2d --workload gradient --steps 3 --no-cpu
bash tools/gpu_prof.sh c1 stencil_kernel --config 1 --steps 5 --warmup 3 --no-e2e --no-cpu

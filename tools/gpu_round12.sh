set -x
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
for w in gradient ingest; do
  python bench.py --workload $w --steps 20 > gpurun_out/bench_r01_$w.json 2> gpurun_out/bench_r01_$w.err || tail -5 gpurun_out/bench_r01_$w.err
  python3 -c "
import json;d=json.load(open('gpurun_out/bench_r01_$w.json'));print('$w',d['ms_per_step'],json.dumps(d['roofline'])[:200]);print(' cpu',d['cpu_baseline']['value']);print(' e2e',d['e2e'])"
done

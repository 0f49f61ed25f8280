timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "lcp or LCP or boundary" > gpurun_out/alltest.txt 2>&1
for w in lcp lcpfused; do timeout 300 python bench.py --workload $w --steps 20 --no-cpu > gpurun_out/w_$w.json 2>gpurun_out/w_$w.err || tail -3 gpurun_out/w_$w.err; done
python -c "
import json
for w in ('lcp','lcpfused'):
    d=json.load(open(f'gpurun_out/w_{w}.json')); print(w, d['ms_per_step'], d['roofline']['frac'])"
tail -1 gpurun_out/alltest.txt

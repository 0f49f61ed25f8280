set -x
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "mc" 2>&1 | tail -5
timeout 300 python bench.py --config 2 --steps 10 --no-cpu > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; tail -3 gpurun_out/bench_c2.err
python3 -c "import json;d=json.load(open('gpurun_out/bench_c2.json'));print(d['ms_per_step'],d['value'],d['e2e'])"

timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/alltest.txt 2>&1
timeout 300 python bench.py --config 3 --steps 20 --no-cpu --no-e2e > gpurun_out/c3.json 2>gpurun_out/c3.err || tail -3 gpurun_out/c3.err
timeout 300 python bench.py --config 0 --steps 50 --no-cpu --no-e2e > gpurun_out/c0.json 2>gpurun_out/c0.err || tail -3 gpurun_out/c0.err
python -c "import json;d=json.load(open('gpurun_out/c3.json'));print('c3',d['ms_per_step'],d['roofline']['frac'],d['fp64_variant']['ms_per_step'],d['fp64_variant']['roofline']['frac']); d=json.load(open('gpurun_out/c0.json')); print('c0', d['ms_per_step'])"
tail -3 gpurun_out/alltest.txt

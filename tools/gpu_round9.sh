timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
python bench.py --config 1 --no-cpu --no-e2e > gpurun_out/bench_c1.json 2>&1; grep -o '"ms_per_step": [0-9.]*' gpurun_out/bench_c1.json; grep -o '"frac": [0-9.]*' gpurun_out/bench_c1.json

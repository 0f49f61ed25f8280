python -c "import __graft_entry__ as g; print('stale on box:', g._stale())"
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
python bench.py --config 2 --no-cpu --no-e2e --steps 10 > gpurun_out/bench_c2.json 2>&1; grep -o '"ms_per_step": [0-9.]*' gpurun_out/bench_c2.json

timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
python bench.py --config 4 --no-cpu --no-e2e --steps 10 --warmup 3 > gpurun_out/bench_c4.json 2>&1; cut -c1-400 gpurun_out/bench_c4.json; grep -o '"roofline": {[^}]*}' gpurun_out/bench_c4.json
bash tools/gpu_prof.sh k3v1 k3_tma --config 4 --no-cpu --no-e2e --steps 3 --warmup 3

timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "ensemble" 2>&1 | tail -2
python bench.py --config 4 --no-cpu --no-e2e --steps 20 --warmup 3 > gpurun_out/bench_c4.json 2>&1; grep -o '"ms_per_step": [0-9.]*' gpurun_out/bench_c4.json; grep -o '"frac": [0-9.]*' gpurun_out/bench_c4.json
bash tools/gpu_prof.sh k3v2 k3_tma --config 4 --no-cpu --no-e2e --steps 3 --warmup 3

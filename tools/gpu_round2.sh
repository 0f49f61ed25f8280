set -x
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -15
python bench.py --no-cpu > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -3 gpurun_out/bench_c3.err
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k2_tma -s 3 -c 1 -o gpurun_out/prof_k2tma_c3 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu2.log 2>&1
cat gpurun_out/bench_c3.json

set -x
python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -3 gpurun_out/bench_c3.err
python bench.py --config 1 --no-cpu > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; tail -3 gpurun_out/bench_c1.err
python bench.py --config 4 --no-cpu --no-e2e --steps 20 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; tail -3 gpurun_out/bench_c4.err
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:stencil_kernel -s 3 -c 1 -o gpurun_out/prof_k2_c3 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu2.log 2>&1
python bench.py --config 4 --no-cpu --no-e2e --steps 5 --warmup 3 > gpurun_out/plain4.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:stencil_kernel -s 3 -c 1 -o gpurun_out/prof_k3_c4 python bench.py --config 4 --no-cpu --no-e2e --steps 5 --warmup 3 > gpurun_out/ncu3.log 2>&1
cat gpurun_out/bench_c3.json gpurun_out/bench_c1.json gpurun_out/bench_c4.json

timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
for c in 3 4 1 0 2; do
  extra=""; [ $c = 4 ] && extra="--no-e2e --steps 20"; [ $c = 2 ] && extra="--steps 5"
  python bench.py --config $c $extra > gpurun_out/bench_r01_c$c.json 2> gpurun_out/bench_r01_c$c.err || tail -5 gpurun_out/bench_r01_c$c.err
done
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_r01_ref.json 2>&1
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,memory.total --format=csv > gpurun_out/gpuinfo.csv; lscpu | grep -E "Model name|^CPU\(s\)|Socket" >> gpurun_out/gpuinfo.csv

set -x
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
for w in lcp gradient ingest; do
  python bench.py --workload $w --steps 20 > gpurun_out/bench_r01_$w.json 2> gpurun_out/bench_r01_$w.err || tail -5 gpurun_out/bench_r01_$w.err
  cut -c1-600 gpurun_out/bench_r01_$w.json
done
python bench.py --workload lcp --steps 3 --no-cpu > gpurun_out/plain_lcp.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:lcp2d --csv --log-file gpurun_out/launches_lcp.csv python bench.py --workload lcp --steps 3 --no-cpu > gpurun_out/ncu_lcp.log 2>&1
python bench.py --workload gradient --steps 3 --no-cpu > gpurun_out/plain_gr.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:gradient2d --csv --log-file gpurun_out/launches_gradient.csv python bench.py --workload gradient --steps 3 --no-cpu > gpurun_out/ncu_gr.log 2>&1

# Round profiles: launch lists of the default bench + one --set full capture per hot kernel.
set -x
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_config3.csv \
  python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
python bench.py --config 4 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain4.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_config4.csv \
  python bench.py --config 4 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch4.log 2>&1
bash tools/gpu_prof.sh k2 k2_tma --config 3 --steps 5 --warmup 3 --no-e2e --no-cpu
bash tools/gpu_prof.sh k3 k3_tma --config 4 --steps 3 --warmup 3 --no-e2e --no-cpu
bash tools/gpu_prof.sh c1 k3_tma --config 1 --steps 5 --warmup 3 --no-e2e --no-cpu
bash tools/gpu_prof.sh mc mc_chunk --config 2 --steps 3 --warmup 3 --no-e2e --no-cpu
bash tools/gpu_prof.sh lcp lcp2d --workload lcp --steps 3 --no-cpu --no-e2e
bash tools/gpu_prof.sh gradient gradient2d --workload gradient --steps 3 --no-cpu --no-e2e
bash tools/gpu_prof.sh fit fit_stream --workload fit --steps 3 --no-cpu --no-e2e
ls -la gpurun_out/*.ncu-rep

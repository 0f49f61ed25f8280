# Round profiles: launch lists of the default bench + one --set full capture per hot kernel.
# Summaries are written on the box; only the K2 / K3 reports are kept (gpurun_out <= 64 MiB).
set -x
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_config3.csv \
  python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
python bench.py --config 4 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain4.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_config4.csv \
  python bench.py --config 4 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch4.log 2>&1
prof() {  # name kernel-regex bench-args...
  name=$1; shift; kre=$1; shift
  bash tools/gpu_prof.sh $name $kre "$@"
  python tools/ncu_summary.py gpurun_out/prof_$name.ncu-rep > gpurun_out/sum_$name.txt
}
prof k2 k2_tma --config 3 --steps 5 --warmup 3 --no-e2e --no-cpu
prof k3 k3_tma --config 4 --steps 3 --warmup 3 --no-e2e --no-cpu
prof c1 k3_rowmarch --config 1 --steps 5 --warmup 3 --no-e2e --no-cpu
prof mc mc_chunk --config 2 --steps 3 --warmup 3 --no-e2e --no-cpu
prof lcp lcp2d_tma --workload lcp --steps 3 --no-cpu --no-e2e
prof gradient gradient_tma --workload gradient --steps 3 --no-cpu --no-e2e
prof fit fit_bulk --workload fit --steps 3 --no-cpu --no-e2e
prof redsea gradfused --workload redsea --steps 3 --no-cpu --no-e2e
rm -f gpurun_out/prof_c1.ncu-rep gpurun_out/prof_mc.ncu-rep gpurun_out/prof_lcp.ncu-rep \
      gpurun_out/prof_gradient.ncu-rep gpurun_out/prof_fit.ncu-rep gpurun_out/prof_redsea.ncu-rep
du -sh gpurun_out

# ncu evidence at the final HEAD of round 2: launch lists of the bench commands
# and one `ncu --set full` capture per hot kernel (summaries + SASS mix kept).
# Output: gpurun_out/r02f/ (copied into profiles/r02b/).
O=gpurun_out/r02f
mkdir -p $O
launch() {  # name, bench args...
  n=$1; shift
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$n.csv \
    python bench.py "$@" --no-e2e --no-cpu --no-fp64 > /dev/null 2>&1
}
launch config3 --config 3 --steps 5 --warmup 3
launch config4 --config 4 --steps 3 --warmup 3
launch config1 --config 1 --steps 5 --warmup 3
launch config2 --config 2 --steps 3 --warmup 3
launch lcp --workload lcp --steps 3 --warmup 3
launch redsea --workload redsea --steps 3 --warmup 3
prof() {  # name kernel-regex bench-args...
  n=$1; shift; k=$1; shift
  ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o $O/prof_$n \
    python bench.py "$@" --no-e2e --no-cpu --no-fp64 > $O/ncu_$n.log 2>&1
  python tools/ncu_summary.py $O/prof_$n.ncu-rep > $O/${n}_summary.txt
  ncu -i $O/prof_$n.ncu-rep --page source --csv --print-source sass > $O/src_$n.csv 2>/dev/null
  python tools/sass_mix_csv.py $O/src_$n.csv > $O/${n}_sassmix.txt 2>/dev/null
  rm -f $O/prof_$n.ncu-rep $O/src_$n.csv
}
prof k2_tma_config3 k2_tma --config 3 --steps 5 --warmup 3
prof k3_tma_config4slab k3_tma --config 4 --steps 3 --warmup 3
prof k3_rowmarch_config1 k3_rowmarch --config 1 --steps 5 --warmup 3
prof mc_chunk_config2 mc_chunk --config 2 --steps 3 --warmup 3
prof gradfused_redsea gradfused --workload redsea --steps 3
prof fit_bulk fit_bulk --workload fit --steps 3
prof gradient_tma gradient_tma --workload gradient --steps 3
ls $O

# Pipe-utilisation captures for the compute-bound kernels (scratch tool).
O=gpurun_out/pipes
mkdir -p $O
prof() {  # name kernel-regex bench-args...
  n=$1; shift; k=$1; shift
  ncu --set full --clock-control none -k regex:$k -s 3 -c 1 -o $O/prof_$n \
    python bench.py "$@" --no-e2e --no-cpu --no-fp64 > $O/ncu_$n.log 2>&1
  ncu -i $O/prof_$n.ncu-rep --page raw --csv > $O/raw_$n.csv 2>/dev/null
  rm -f $O/prof_$n.ncu-rep
}
prof mc mc_chunk --config 2 --steps 3 --warmup 3
prof lcp lcp2d_tma --workload lcp --steps 3
prof gf gradfused --workload redsea --steps 3
ls -la $O

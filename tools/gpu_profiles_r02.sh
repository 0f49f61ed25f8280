# Round-2 evidence on one B200: GPU tests, every bench line (ours + reference
# arm), ncu launch lists of the bench commands, one `ncu --set full` capture
# per hot kernel (summaries + per-opcode SASS mix kept, reports dropped).
# Output: gpurun_out/r02/ (copied into profiles/r02/ by hand after review).
O=gpurun_out/r02
mkdir -p $O
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,memory.total,power.limit --format=csv > $O/box.txt
lscpu | grep -E "Model name|^CPU\(s\)|Socket" >> $O/box.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gpu_tests.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
: > $O/bench_lines.jsonl
run() {  # name, args...
  n=$1; shift
  timeout 900 python bench.py "$@" > $O/bench_$n.json 2> $O/bench_$n.err && cat $O/bench_$n.json >> $O/bench_lines.jsonl
}
run config3 --config 3
run config4 --config 4 --steps 20
run config1 --config 1
run config0 --config 0
run config2 --config 2 --steps 20
for w in lcp lcpfused gradient fit redsea ingest; do run $w --workload $w --steps 20; done
for c in 3 0 1 2 4; do run ref$c --impl reference --config $c --steps 10 --warmup 3; done
launch() {  # name, bench args...
  n=$1; shift
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$n.csv \
    python bench.py "$@" --no-e2e --no-cpu --no-fp64 > /dev/null 2>&1
}
launch config3 --config 3 --steps 5 --warmup 3
launch config4 --config 4 --steps 3 --warmup 3
launch config1 --config 1 --steps 5 --warmup 3
launch lcpfused --workload lcpfused --steps 3 --warmup 3
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
prof lcp2d_tma lcp2d_tma --workload lcp --steps 3
prof lcp2d_fused lcp2d_fused --workload lcpfused --steps 3
prof gradfused_redsea gradfused --workload redsea --steps 3
prof fit_bulk fit_bulk --workload fit --steps 3
prof gradient_tma gradient_tma --workload gradient --steps 3
# the fp64 K2 of config 3's fp64 side line (launched after the fp32 timed loop)
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"k2_tma_kernel<double" -s 3 -c 1 -o $O/prof_k2_tma_f64 \
  python bench.py --config 3 --steps 3 --warmup 3 --no-e2e --no-cpu > $O/ncu_k2_tma_f64.log 2>&1
python tools/ncu_summary.py $O/prof_k2_tma_f64.ncu-rep > $O/k2_tma_f64_summary.txt
ncu -i $O/prof_k2_tma_f64.ncu-rep --page source --csv --print-source sass > $O/src_k2f64.csv 2>/dev/null
python tools/sass_mix_csv.py $O/src_k2f64.csv > $O/k2_tma_f64_sassmix.txt 2>/dev/null
rm -f $O/prof_k2_tma_f64.ncu-rep $O/src_k2f64.csv
ls -la $O
python tools/dropin_probe.py > $O/dropin_probe.txt 2>&1

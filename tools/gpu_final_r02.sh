# End-of-round check at HEAD: GPU tests, smoke, the default bench line and the
# LCP lines (the kernels changed last) -> gpurun_out/r02d/
O=gpurun_out/r02d
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gpu_tests.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/smoke.txt
: > $O/bench_lines.jsonl
run() { n=$1; shift; timeout 900 python bench.py "$@" > $O/bench_$n.json 2> $O/bench_$n.err && cat $O/bench_$n.json >> $O/bench_lines.jsonl; }
run config3
run lcp --workload lcp --steps 20
run lcpfused --workload lcpfused --steps 20
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_lcpfused.csv \
  python bench.py --workload lcpfused --steps 3 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
tail -1 $O/gpu_tests.txt; cat $O/smoke.txt

# Late-round-2 refresh on one B200 (kernels unchanged since the ncu captures in
# profiles/r02): GPU tests, smoke, every bench line (ours + reference arm),
# drop-in / host-path probes.  Output: gpurun_out/r02c/.
O=gpurun_out/r02c
mkdir -p $O
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,memory.total,power.limit --format=csv > $O/box.txt
lscpu | grep -E "Model name|^CPU\(s\)|Socket" >> $O/box.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gpu_tests.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/smoke.txt
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
timeout 900 python tools/dropin_probe.py > $O/dropin_probe.txt 2>&1
timeout 600 python tools/bounce_probe.py > $O/bounce_probe.txt 2>&1
timeout 600 python tools/device_call_probe.py > $O/device_call_probe.txt 2>&1
timeout 600 python tools/host_entry_trace.py 128 > $O/host_entry_trace.txt 2>&1
ls -la $O
timeout 600 python tools/fit_trace.py 2>&1 | grep -E "ms, all" > $O/fit_trace.txt

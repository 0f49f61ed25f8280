python -c "import __graft_entry__ as g; g.build()"
FLUSH=write python tools/sweep_c1.py
FLUSH=drain python tools/sweep_c1.py
FLUSH=drain SWEEP="DIVUQ_NO_TMA=0,1" python tools/sweep_c1.py
python bench.py --config 1 --no-cpu > gpurun_out/bench_c1.json; cut -c1-300 gpurun_out/bench_c1.json
python bench.py --config 0 --no-cpu > gpurun_out/bench_c0.json; cut -c1-300 gpurun_out/bench_c0.json

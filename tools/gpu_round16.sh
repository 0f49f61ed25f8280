python -c "import __graft_entry__ as g; g.build()"
SWEEP="DIVUQ_K3_HDELAY=0,1,2,3" python tools/sweep_c1.py
C1_N=2048 SWEEP="DIVUQ_K3_HDELAY=0,1,2,3" python tools/sweep_c1.py
C1_N=4096 C1_M=10 SWEEP="DIVUQ_K3_HDELAY=0,1,3" python tools/sweep_c1.py
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "ensemble or fused or k3 or tma" 2>&1 | tail -2
python bench.py --config 4 --no-cpu --no-e2e --steps 20 > gpurun_out/bench_c4.json 2>&1; grep -o '"ms_per_step": [0-9.]*' gpurun_out/bench_c4.json

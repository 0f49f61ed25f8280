python -c "import __graft_entry__ as g; g.build()"
python tools/sweep_c1.py
SWEEP="DIVUQ_TMA_PROMO=0,128,256" python tools/sweep_c1.py
C1_N=2048 python tools/sweep_c1.py
bash tools/gpu_prof.sh c1 k3_tma --config 1 --steps 5 --warmup 3 --no-e2e --no-cpu
python tools/ncu_summary.py gpurun_out/prof_c1.ncu-rep > gpurun_out/sum_c1.txt 2>&1

timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -5
SWEEP_PROMO=256,0 SWEEP_TY=0,16 python tools/sweep_k2.py
bash tools/gpu_prof.sh k2v6 k2_tma --steps 5 --warmup 3 --no-e2e --no-cpu

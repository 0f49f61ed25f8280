timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -5
SWEEP_PROMO=256 SWEEP_TY=0,16,8 python tools/sweep_k2.py

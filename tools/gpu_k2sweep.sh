timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "3d or k2 or slab or shard or fullsize or propagate" 2>&1 | tail -3
SWEEP="DIVUQ_K2_SYNC_W=0,8;DIVUQ_K2_HDELAY=1,2" python tools/sweep_k2.py 2>&1 | tail -4

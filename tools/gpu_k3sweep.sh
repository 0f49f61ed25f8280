SWEEP="DIVUQ_K3_SYNC_W=0,2,4;DIVUQ_K3_HDELAY=0,1,2" python tools/sweep_k3.py 2>&1 | tail -9
K3_NZL=64 SWEEP="DIVUQ_K3_SYNC_W=0,2;DIVUQ_K3_HDELAY=1,2" python tools/sweep_k3.py 2>&1 | tail -4

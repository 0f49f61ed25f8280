SWEEP="DIVUQ_TMA_TY=0,16,12" python tools/sweep_k2.py
SWEEP="DIVUQ_NO_TMA=0,1" python tools/sweep_k2.py

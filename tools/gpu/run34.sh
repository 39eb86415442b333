python tools/kbench.py --B 1024 --T 500 --tag "c2 K2" 2>&1 | tail -2
LCB_RESIDENT=0 python tools/kbench.py --B 1024 --T 500 --tag "c2 K1s" 2>&1 | tail -2

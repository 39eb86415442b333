for n in 2000 5000 10000; do
for B in 256 1024; do
python tools/kbench.py --n $n --B $B --T 300 --quco-only --tag "n=$n K2" 2>&1 | tail -1
LCB_RESIDENT=0 python tools/kbench.py --n $n --B $B --T 300 --quco-only --tag "n=$n K1s" 2>&1 | tail -1
done
done
python tools/kbench.py --B 1024 --T 200 --precision fp64 --tag "c2 fp64 K2" 2>&1 | tail -2
LCB_RESIDENT=0 python tools/kbench.py --B 1024 --T 200 --precision fp64 --tag "c2 fp64 K1s" 2>&1 | tail -2

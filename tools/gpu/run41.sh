for prec in fp32 fp64; do
for n in 2000 5000 10000; do
for B in 256 1024; do
python tools/kbench.py --n $n --B $B --T 300 --precision $prec --tag "$prec n=$n B=$B K2" 2>&1 | tail -2
LCB_RESIDENT=0 python tools/kbench.py --n $n --B $B --T 300 --precision $prec --tag "$prec n=$n B=$B K1s" 2>&1 | tail -2
done
done
done

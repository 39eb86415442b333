for n in 5000 10000; do
for B in 256 1024; do
LCB_BANK_ORDER=0 python tools/kbench.py --n $n --B $B --T 300 --tag "fp32 n=$n B=$B K2-csr" 2>&1 | tail -2
done
done

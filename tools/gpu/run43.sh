export LCB_LIB_PATH=build_variants/seq.so
for B in 128 256 512 1024; do
LCB_BANK_ORDER=0 python tools/kbench.py --B $B --T 300 --tag "c2 K2-seq-csr B=$B" 2>&1 | tail -2
done
unset LCB_LIB_PATH
for B in 128 256 512; do
LCB_RESIDENT=0 python tools/kbench.py --B $B --T 300 --tag "c2 K1s B=$B" 2>&1 | tail -2
done

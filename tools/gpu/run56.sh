nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv
for v in head cache head cache; do
export LCB_LIB_PATH=build_variants/$v.so
python tools/kbench.py --B 1024 --T 500 --tag "c2 $v" 2>&1 | tail -2
done

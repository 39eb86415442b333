for v in default fnb1 fnb4; do
if [ $v = default ]; then unset LCB_LIB_PATH; else export LCB_LIB_PATH=build_variants/$v.so; fi
python tools/kbench.py --graph er --n 1000000 --B 512 --T 20 --quco-only --tag "c4 T20 $v" 2>&1 | tail -1
python tools/kbench.py --graph er --n 1000000 --B 512 --T 500 --quco-only --tag "c4 $v" 2>&1 | tail -1
done

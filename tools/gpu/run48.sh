for v in default fnb1; do
if [ $v = default ]; then unset LCB_LIB_PATH; else export LCB_LIB_PATH=build_variants/$v.so; fi
python tools/kbench.py --graph ba --n 100000 --B 256 --T 500 --quco-only --tag "c5 $v" 2>&1 | tail -1
python tools/kbench.py --graph er --n 1000000 --B 512 --T 200 --quco-only --precision fp64 --tag "c4 fp64 $v" 2>&1 | tail -1
python tools/kbench.py --B 1024 --T 200 --precision fp64 --tag "c2 fp64 $v" 2>&1 | tail -2
python tools/kbench.py --graph er --n 1000000 --B 512 --T 500 --quco-only --tag "c4 $v" 2>&1 | tail -1
done

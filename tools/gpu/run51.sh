for v in default f64n1 f64n3 f64n4; do
if [ $v = default ]; then unset LCB_LIB_PATH; else export LCB_LIB_PATH=build_variants/$v.so; fi
python tools/kbench.py --graph er --n 1000000 --B 512 --T 200 --quco-only --precision fp64 --tag "c4 fp64 $v" 2>&1 | tail -1
python tools/kbench.py --B 1024 --T 200 --precision fp64 --tag "c2 fp64 $v" 2>&1 | tail -1
done

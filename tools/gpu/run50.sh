for v in default s3 l2 r22 r24 s5; do
if [ $v = default ]; then unset LCB_LIB_PATH; else export LCB_LIB_PATH=build_variants/$v.so; fi
python tools/kbench.py --graph er --n 1000000 --B 512 --T 500 --quco-only --tag "c4 $v" 2>&1 | tail -1
python tools/kbench.py --graph ba --n 100000 --B 256 --T 500 --quco-only --tag "c5 $v" 2>&1 | tail -1
done

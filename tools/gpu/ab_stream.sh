# K1s correctness + A/B of its variants (one box)
python -m pytest tests/test_gpu_stream.py -x -q 2>&1 | tail -15
for v in s16m2 s16m1 s24m1 s31m1; do
  LCB_LIB_PATH=build_variants/$v.so python tools/kbench.py --graph er --n 1000000 --B 512 --T 100 --quco-only --tag "c4 $v" 2>&1 | tail -1
  LCB_LIB_PATH=build_variants/$v.so python tools/kbench.py --graph ba --n 100000 --B 256 --T 200 --quco-only --tag "c5 $v" 2>&1 | tail -1
  LCB_RESIDENT=0 LCB_LIB_PATH=build_variants/$v.so python tools/kbench.py --graph ba --n 10000 --B 1024 --T 200 --tag "c2 $v" 2>&1 | tail -2
done
LCB_STREAM=0 python tools/kbench.py --graph er --n 1000000 --B 512 --T 100 --quco-only --tag "c4 K1" 2>&1 | tail -1
python tools/kbench.py --graph ba --n 10000 --B 1024 --T 200 --tag "c2 K2" 2>&1 | tail -2

LCB_STREAM=1 timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_kernels_fp32.py -q -x --timeout 600 2>&1 | tail -3
LCB_STREAM=1 python tools/kbench.py --graph er --n 1000000 --B 512 --T 100 --quco-only --tag "c4 fnb4" 2>&1 | tail -1
for v in f2 f8; do LCB_STREAM=1 LCB_LIB_PATH=build_variants/$v.so python tools/kbench.py --graph er --n 1000000 --B 512 --T 100 --quco-only --tag "c4 $v" 2>&1 | tail -1; done
LCB_STREAM=1 python tools/kbench.py --graph ba --n 100000 --B 256 --T 200 --quco-only --tag "c5 fnb4" 2>&1 | tail -1
LCB_STREAM=1 LCB_RESIDENT=0 python tools/kbench.py --graph ba --n 10000 --B 1024 --T 200 --tag "c2 K1s" 2>&1 | tail -2
python tools/kbench.py --graph ba --n 10000 --B 1024 --T 200 --tag "c2 K2" 2>&1 | tail -2

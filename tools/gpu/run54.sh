timeout 1500 python -m pytest tests/test_gpu_stream.py tests/test_gpu_kernels_fp32.py tests/test_gpu_parity.py -q -x --timeout 900 2>&1 | tail -1
for p in 1 0; do
LCB_PAIR=$p python tools/kbench.py --graph er --n 1000000 --B 512 --T 500 --quco-only --tag "c4 pair=$p" 2>&1 | tail -1
LCB_PAIR=$p python tools/kbench.py --graph er --n 1000000 --B 512 --T 200 --quco-only --precision fp64 --tag "c4 fp64 pair=$p" 2>&1 | tail -1
done
python tools/kbench.py --graph ba --n 100000 --B 256 --T 500 --quco-only --tag "c5" 2>&1 | tail -1

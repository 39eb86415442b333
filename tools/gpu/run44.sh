timeout 1500 python -m pytest tests/test_gpu_stream.py tests/test_gpu_kernels_fp32.py tests/test_gpu_parity.py tests/test_gpu_multirank.py -q -x --timeout 900 2>&1 | tail -1
for B in 64 128 200 256; do
LCB_RESIDENT=0 python tools/kbench.py --B $B --T 300 --quco-only --tag "c2 K1s B=$B" 2>&1 | tail -1
done
python tools/kbench.py --graph er --n 1000000 --B 100 --T 100 --quco-only --tag "c4-graph B=100" 2>&1 | tail -1
python tools/kbench.py --graph er --n 1000000 --B 512 --T 500 --quco-only --tag "c4" 2>&1 | tail -1

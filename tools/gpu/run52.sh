timeout 1500 python -m pytest tests/test_gpu_stream.py tests/test_gpu_kernels_fp32.py -q -x --timeout 900 2>&1 | tail -1
python tools/kbench.py --graph er --n 1000000 --B 512 --T 20 --quco-only --tag "c4 T20" 2>&1 | tail -1
python tools/kbench.py --graph er --n 1000000 --B 512 --T 500 --quco-only --tag "c4" 2>&1 | tail -1
python tools/kbench.py --graph ba --n 100000 --B 256 --T 500 --quco-only --tag "c5" 2>&1 | tail -1

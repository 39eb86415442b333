timeout 1500 python -m pytest tests/test_gpu_stream.py tests/test_gpu_kernels_fp32.py -q -x --timeout 900 2>&1 | tail -2
python tools/kbench.py --graph er --n 1000000 --B 512 --T 500 --quco-only --tag "c4" 2>&1 | tail -1
python tools/kbench.py --graph ba --n 100000 --B 256 --T 500 --quco-only --tag "c5" 2>&1 | tail -1
python tools/kbench.py --graph er --n 1000000 --B 512 --T 200 --quco-only --precision fp64 --tag "c4 fp64" 2>&1 | tail -1
python tools/kbench.py --graph er --n 1000000 --B 512 --T 100 --quco-only --tag c4 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -k regex:k_stream -s 690 -c 1 python tools/kbench.py --graph er --n 1000000 --B 512 --T 100 --quco-only --tag c4 2>&1 | grep -E "duration|inst_exec|bytes"

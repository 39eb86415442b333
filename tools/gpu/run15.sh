timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_kernels_fp32.py -q -x --timeout 600 2>&1 | tail -2
python tools/kbench.py --graph ba --n 100000 --B 256 --T 200 --quco-only --tag "c5" 2>&1 | tail -1
python tools/kbench.py --graph er --n 1000000 --B 512 --T 100 --quco-only --tag "c4" 2>&1 | tail -1
python tools/kbench.py --graph ba --n 100000 --B 256 --T 200 --quco-only --tag c5 > gpurun_out/k1s_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_active.avg,sm__cycles_active.max --clock-control none -k regex:k_stream -s 600 -c 200 --csv --log-file gpurun_out/k1s_c5_launches2.csv python tools/kbench.py --graph ba --n 100000 --B 256 --T 200 --quco-only --tag c5 > gpurun_out/k1s_ncu1.log 2>&1
tail -n 1 gpurun_out/k1s_ncu1.log

python -m pytest tests/test_gpu_stream.py tests/test_gpu_multirank.py -x -q 2>&1 | tail -4
for v in w1 w2 w3 w4 w5; do
  LCB_LIB_PATH=build_variants/$v.so python tools/kbench.py --graph er --n 1000000 --B 512 --T 100 --quco-only --tag "c4 $v" 2>&1 | tail -1
  LCB_LIB_PATH=build_variants/$v.so python tools/kbench.py --graph ba --n 100000 --B 256 --T 200 --quco-only --tag "c5 $v" 2>&1 | tail -1
done
LCB_LIB_PATH=build_variants/w1.so python tools/kbench.py --graph er --n 1000000 --B 512 --T 100 --quco-only --tag c4 > gpurun_out/k1s_plain.log 2>&1 && LCB_LIB_PATH=build_variants/w1.so ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -k regex:k_stream -s 1200 -c 400 --csv --log-file gpurun_out/k1s_c4_launches4.csv python tools/kbench.py --graph er --n 1000000 --B 512 --T 100 --quco-only --tag c4 > gpurun_out/k1s_ncu1.log 2>&1
tail -n 1 gpurun_out/k1s_ncu1.log

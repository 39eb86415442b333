python -m pytest tests/test_gpu_stream.py -x -q 2>&1 | tail -3
for v in p4 p8 p4nb16 p4s6; do
  LCB_LIB_PATH=build_variants/$v.so python tools/kbench.py --graph er --n 1000000 --B 512 --T 100 --quco-only --tag "c4 $v" 2>&1 | tail -1
  LCB_LIB_PATH=build_variants/$v.so python tools/kbench.py --graph ba --n 100000 --B 256 --T 200 --quco-only --tag "c5 $v" 2>&1 | tail -1
  LCB_RESIDENT=0 LCB_LIB_PATH=build_variants/$v.so python tools/kbench.py --graph ba --n 10000 --B 1024 --T 200 --quco-only --tag "c2 $v" 2>&1 | tail -1
done
python tools/kbench.py --graph er --n 1000000 --B 512 --T 40 --quco-only --tag c4 > gpurun_out/k1s_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_stream -s 130 -c 1 -o gpurun_out/k1s_c4 python tools/kbench.py --graph er --n 1000000 --B 512 --T 40 --quco-only --tag c4 > gpurun_out/k1s_ncu.log 2>&1
tail -n 2 gpurun_out/k1s_ncu.log

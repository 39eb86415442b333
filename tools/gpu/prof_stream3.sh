python tools/kbench.py --graph er --n 1000000 --B 512 --T 100 --quco-only --tag c4 > gpurun_out/k1s_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_stream -s 1290 -c 1 -o gpurun_out/k1s_c4_sat4 python tools/kbench.py --graph er --n 1000000 --B 512 --T 100 --quco-only --tag c4 > gpurun_out/k1s_ncu2.log 2>&1
tail -n 1 gpurun_out/k1s_ncu2.log

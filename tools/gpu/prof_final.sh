python tools/kbench.py --B 1024 --T 500 --quco-only --tag c2 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:k_resident -s 1 -c 1 -o gpurun_out/fin_k2 python tools/kbench.py --B 1024 --T 500 --quco-only --tag c2 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:k_epilogue -c 1 -o gpurun_out/fin_k4 python tools/kbench.py --graph er --n 1000000 --B 512 --T 5 --quco-only --tag c4 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:k_dense_step -s 40 -c 1 -o gpurun_out/fin_k3 python tools/prof_dense.py --T 30 > /dev/null 2>&1
ls gpurun_out/fin_*

python tools/kbench.py --graph er --n 1000000 --B 512 --T 100 --quco-only --tag c4 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_stream -s 690 -c 1 -o gpurun_out/r23_c4_sat python tools/kbench.py --graph er --n 1000000 --B 512 --T 100 --quco-only --tag c4 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_stream -s 605 -c 1 -o gpurun_out/r23_c4_unsat python tools/kbench.py --graph er --n 1000000 --B 512 --T 100 --quco-only --tag c4 > /dev/null 2>&1
ls gpurun_out | grep r23

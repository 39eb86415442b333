ncu --set full --clock-control none -k regex:k_epilogue -c 1 -o gpurun_out/c3_epi python tools/prof_dense.py --T 3 > /dev/null 2>&1; ls gpurun_out/c3_epi.ncu-rep

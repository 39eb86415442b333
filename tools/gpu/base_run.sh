set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python tools/kbench.py --graph er --n 1000000 --B 512 --T 40 --quco-only --tag c4 > gpurun_out/base_kb_c4.log 2>&1
python tools/kbench.py --graph ba --n 100000 --B 256 --T 100 --quco-only --tag c5 > gpurun_out/base_kb_c5.log 2>&1
cat gpurun_out/base_kb_c4.log gpurun_out/base_kb_c5.log
ncu --set full --clock-control none --import-source on -k regex:k_step -s 100 -c 2 -o gpurun_out/base_k1_c4 python tools/kbench.py --graph er --n 1000000 --B 512 --T 40 --quco-only --tag c4 > gpurun_out/base_ncu_c4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_step -s 250 -c 2 -o gpurun_out/base_k1_c5 python tools/kbench.py --graph ba --n 100000 --B 256 --T 100 --quco-only --tag c5 > gpurun_out/base_ncu_c5.log 2>&1
tail -3 gpurun_out/base_ncu_c4.log gpurun_out/base_ncu_c5.log

timeout 900 python -m pytest tests/test_gpu_stream.py -q -x --timeout 900 2>&1 | tail -1
for v in default e1 e1n8 e1n8s e1n8c4 n8 n8c4; do
if [ $v = default ]; then unset LCB_LIB_PATH; else export LCB_LIB_PATH=build_variants/$v.so; fi
python tools/kbench.py --graph er --n 1000000 --B 512 --T 500 --quco-only --tag "c4 $v" 2>&1 | tail -1
done
unset LCB_LIB_PATH
python tools/kbench.py --graph er --n 1000000 --B 512 --T 100 --quco-only --tag c4 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_stream -s 690 -c 1 -o gpurun_out/fp_c4_sat python tools/kbench.py --graph er --n 1000000 --B 512 --T 100 --quco-only --tag c4 > /dev/null 2>&1; ls gpurun_out/

timeout 1500 python -m pytest tests/test_gpu_kernels_fp32.py tests/test_gpu_parity.py tests/test_gpu_dense.py -q -x --timeout 900 2>&1 | tail -1
for v in default nocache; do
if [ $v = default ]; then unset LCB_LIB_PATH; else export LCB_LIB_PATH=build_variants/$v.so; fi
python tools/kbench.py --B 1024 --T 500 --tag "c2 $v" 2>&1 | tail -2
python tools/kbench.py --n 5000 --B 256 --T 300 --tag "n5k $v" 2>&1 | tail -2
done

timeout 1500 python -m pytest tests/test_gpu_objectives.py tests/test_gpu_dense.py tests/test_gpu_parity.py -q -x --timeout 900 2>&1 | tail -1
python tools/gpu/c3_stages.py 2>&1 | tail -2

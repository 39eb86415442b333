timeout 600 python -m pytest tests/test_gpu_multirank.py -q -x --timeout 300 -k search 2>&1 | grep -E "^(E|>|tests/|paper)" | head -30
LCB_STREAM=0 timeout 600 python -m pytest tests/test_gpu_multirank.py -q -x --timeout 300 -k search 2>&1 | tail -2
LCB_SLAB_OUTER=1 timeout 600 python -m pytest tests/test_gpu_multirank.py -q -x --timeout 300 -k search 2>&1 | tail -2

LCB_STREAM=1 timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_kernels_fp32.py tests/test_gpu_objectives.py -q -x --timeout 600 2>&1 | tail -3
LCB_STREAM=1 python tools/kbench.py --graph ba --n 100000 --B 256 --T 200 --quco-only --tag "c5 iter-outer" 2>&1 | tail -1
LCB_STREAM=1 LCB_SLAB_OUTER=1 python tools/kbench.py --graph ba --n 100000 --B 256 --T 200 --quco-only --tag "c5 slab-outer" 2>&1 | tail -1
LCB_STREAM=0 python tools/kbench.py --graph ba --n 100000 --B 256 --T 200 --quco-only --tag "c5 K1" 2>&1 | tail -1
LCB_STREAM=1 LCB_RESIDENT=0 python tools/kbench.py --graph ba --n 10000 --B 1024 --T 200 --tag "c2 K1s" 2>&1 | tail -2
LCB_STREAM=1 python bench.py --config c4 --steps 3 --warmup 3 --no-extras > gpurun_out/bench_c4_k1s.json 2> gpurun_out/bench_c4_k1s.err; tail -c 600 gpurun_out/bench_c4_k1s.json

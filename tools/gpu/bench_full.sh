start=$(date +%s)
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
echo "rc=$? wall=$(( $(date +%s) - start ))s"
tail -c 4000 gpurun_out/bench_full.json
python tools/cut_parity.py > gpurun_out/cut_parity.json 2> gpurun_out/cut_parity.err
echo "cut parity rc=$?"; tail -c 2000 gpurun_out/cut_parity.json

M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum
python tools/kbench.py --graph er --n 1000000 --B 512 --T 100 --quco-only --tag c4 > gpurun_out/tr_plain.log 2>&1 || exit 1
ncu --metrics $M --clock-control none -k regex:k_stream -s 600 -c 200 --csv --log-file gpurun_out/tr_c4_fp32.csv python tools/kbench.py --graph er --n 1000000 --B 512 --T 100 --quco-only --tag c4 > /dev/null 2>&1
ncu --metrics $M --clock-control none -k regex:k_stream -s 1200 -c 400 --csv --log-file gpurun_out/tr_c4_fp64.csv python tools/kbench.py --graph er --n 1000000 --B 512 --T 100 --quco-only --precision fp64 --tag c4 > /dev/null 2>&1
ncu --metrics $M --clock-control none -k regex:k_stream -s 1500 -c 500 --csv --log-file gpurun_out/tr_c5_fp32.csv python tools/kbench.py --graph ba --n 100000 --B 256 --T 500 --quco-only --tag c5 > /dev/null 2>&1
gzip -f gpurun_out/tr_*.csv; ls -la gpurun_out/tr_*

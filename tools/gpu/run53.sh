python tools/kbench.py --graph er --n 1000000 --B 512 --T 100 --quco-only --tag c4 > /dev/null 2>&1
for v in default exp4; do
if [ $v = default ]; then unset LCB_LIB_PATH; else export LCB_LIB_PATH=build_variants/$v.so; fi
echo $v
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:k_stream -s 680 -c 3 python tools/kbench.py --graph er --n 1000000 --B 512 --T 100 --quco-only --tag c4 2>&1 | grep -E "duration|inst_exec"
done

for v in default u8; do
if [ $v = default ]; then unset LCB_LIB_PATH; else export LCB_LIB_PATH=build_variants/$v.so; fi
echo $v; python tools/gpu/c3_stages.py 2>&1 | tail -1 | cut -c1-140
done

mkdir -p gpurun_out
for v in noast nomma both; do
  SMX_LIB_PATH=profiles/debug/var/libsmx_$v.so timeout 300 python profiles/debug/ab_conv1.py 2>&1 | sed "s/^/$v /" >> gpurun_out/ab_c1var.txt
done
cat gpurun_out/ab_c1var.txt

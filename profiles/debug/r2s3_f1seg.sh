for v in f1s1 f1s2 base; do
  if [ $v = base ]; then L=""; else L="SMX_LIB_PATH=profiles/debug/var/libsmx_$v.so"; fi
  echo "== $v"
  env $L timeout 900 python -m pytest tests/test_cnn_gpu.py -q -p no:cacheprovider -k first_step 2>&1 | grep -E "Error: \(|passed|failed"
  env $L timeout 300 python profiles/debug/ab_conv1.py 2>&1 | tail -1
done

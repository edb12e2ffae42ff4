for v in f1noast f1nomma f1nost; do
  SMX_LIB_PATH=profiles/debug/var/libsmx_$v.so timeout 300 python profiles/debug/ab_conv1.py 2>&1 | sed "s/^/$v /"
done

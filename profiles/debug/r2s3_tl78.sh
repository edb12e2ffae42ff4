mkdir -p gpurun_out
V=$PWD/profiles/debug/var
timeout 600 python -m pytest tests/test_cnn_gpu.py tests/test_headline_gpu.py -x -q -p no:cacheprovider --timeout 180 2>&1 | grep -E "passed|failed|Error|assert" | head -20
for lib in TL7 TL8; do SMX_LIB_PATH=$V/libsmx_$lib.so timeout 300 python profiles/debug/timeline.py 4 > gpurun_out/timeline_$lib.txt 2>&1; echo $lib; tail -4 gpurun_out/timeline_$lib.txt | cut -c1-300; done
timeout 600 python profiles/debug/kbench.py $V/libsmx_NEW7.so $V/libsmx_NEW8.so $V/libsmx_NEW7.so $V/libsmx_NEW8.so

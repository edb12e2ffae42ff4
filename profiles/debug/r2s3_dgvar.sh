# conv2 input gradient: A/B of library builds (alternated) + a per-chunk timeline of one CTA
mkdir -p gpurun_out
V=profiles/debug/var
timeout 900 python -m pytest tests/test_cnn_gpu.py tests/test_headline_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -1
timeout 600 python profiles/debug/kbench.py $V/libsmx_NEW.so $V/libsmx_NEW4.so $V/libsmx_NEW.so $V/libsmx_NEW4.so $V/libsmx_NEW.so $V/libsmx_NEW4.so
#SMX_LIB_PATH=$PWD/$V/libsmx_TIMELINE.so timeout 300 python profiles/debug/timeline.py 4 > gpurun_out/timeline_dgrad2.txt 2>&1
#tail -5 gpurun_out/timeline_dgrad2.txt

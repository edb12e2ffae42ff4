mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_cnn_gpu.py tests/test_headline_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -1
bash profiles/debug/r2s3_abk.sh

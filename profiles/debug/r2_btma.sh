timeout 300 python -m pytest tests/test_cnn_gpu.py -q -p no:cacheprovider -x -k "tc_first_step" 2>&1 | tail -5
timeout 300 python -m pytest tests/test_cnn_gpu.py tests/test_headline_gpu.py -q -p no:cacheprovider -x 2>&1 | tail -5
timeout 120 python profiles/debug/ab_kernels.py . 2>&1 | tail -2

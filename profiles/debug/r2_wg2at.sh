mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_cnn_gpu.py tests/test_headline_gpu.py -q -p no:cacheprovider -x 2>&1 | tail -15
timeout 200 python profiles/debug/ab_kernels.py . 2>&1 | tail -3

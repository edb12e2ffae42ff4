mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_cnn_gpu.py tests/test_headline_gpu.py -x -q -p no:cacheprovider > gpurun_out/pytest_c1.txt 2>&1; echo pytest rc $? >> gpurun_out/pytest_c1.txt
timeout 300 python profiles/debug/ab_conv1.py > gpurun_out/ab_c1.txt 2>&1
SMX_CONV1_FWD_LANE=1 SMX_CONV1_WGRAD_LANE=1 timeout 300 python profiles/debug/ab_conv1.py >> gpurun_out/ab_c1.txt 2>&1
tail -15 gpurun_out/pytest_c1.txt; cat gpurun_out/ab_c1.txt

mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_executor_gpu.py tests/test_tuner_gpu.py -x -q -p no:cacheprovider > gpurun_out/pytest_fork.txt 2>&1; echo pytest rc $? >> gpurun_out/pytest_fork.txt
timeout 600 python profiles/occupancy_sweep.py > gpurun_out/occupancy.txt 2>&1
tail -3 gpurun_out/pytest_fork.txt; cat gpurun_out/occupancy.txt

mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; echo pytest rc $? >> gpurun_out/pytest_gpu.txt
timeout 200 python profiles/debug/ab_kernels.py . > gpurun_out/ab.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench.txt 2> gpurun_out/bench.err
tail -3 gpurun_out/pytest_gpu.txt; cat gpurun_out/ab.txt; tail -c 600 gpurun_out/bench.txt

# round-2 session-3 health check: full GPU suite, smoke, default bench, bench launch list
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; echo pytest rc $? >> gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo smoke rc $? >> gpurun_out/smoke.txt
timeout 900 python bench.py > gpurun_out/bench.txt 2> gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 2000 -c 2000 --csv --log-file gpurun_out/bench_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-trial > gpurun_out/bench_ncu.log 2>&1
tail -3 gpurun_out/pytest_gpu.txt; tail -2 gpurun_out/smoke.txt; tail -c 800 gpurun_out/bench.txt

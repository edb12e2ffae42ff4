mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_cnn_gpu.py tests/test_headline_gpu.py -x -q -p no:cacheprovider > gpurun_out/pytest_q.txt 2>&1; echo pytest rc $? >> gpurun_out/pytest_q.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_h.csv python profiles/lockstep_probe.py --model cnn --steps 2 --warmup 1 --bs 128 --max-batch 128 > /dev/null 2>&1
tail -3 gpurun_out/pytest_q.txt; python profiles/launches.py gpurun_out/launches_h.csv 15

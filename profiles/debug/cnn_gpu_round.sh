mkdir -p gpurun_out
timeout 180 python -m pytest tests/test_cnn_gpu.py -q > gpurun_out/pytest_cnn.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_cnn.txt
timeout 120 python profiles/debug/cnn_grad_diag.py > gpurun_out/diag.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cnn_launches.csv python profiles/lockstep_probe.py --model cnn --steps 1 --warmup 1 > /dev/null 2>&1

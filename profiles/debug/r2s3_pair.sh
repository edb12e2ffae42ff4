mkdir -p gpurun_out
timeout 240 python -m pytest tests/test_cnn_gpu.py -x -q -p no:cacheprovider -k "first_step_gradient and not max_batch" > gpurun_out/pair_t1.txt 2>&1; echo "rc $?" >> gpurun_out/pair_t1.txt
tail -3 gpurun_out/pair_t1.txt
grep -E "^E  " gpurun_out/pair_t1.txt | head -5
timeout 300 python profiles/debug/ab_conv1.py 2>&1 | tail -2
SMX_NO_WG3_PAIR=1 timeout 300 python profiles/debug/ab_conv1.py 2>&1 | tail -1

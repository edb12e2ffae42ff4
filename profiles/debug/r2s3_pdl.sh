mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_cnn_gpu.py tests/test_headline_gpu.py tests/test_engine_gpu.py -x -q -p no:cacheprovider > gpurun_out/pytest_q.txt 2>&1; echo pytest rc $? >> gpurun_out/pytest_q.txt
timeout 300 python profiles/occupancy_sweep.py --counts 8,16,34,64 > gpurun_out/occ_pdl.txt 2>&1
SMX_NO_PDL=1 timeout 300 python profiles/occupancy_sweep.py --counts 8,16,34,64 > gpurun_out/occ_nopdl.txt 2>&1
timeout 300 python profiles/occupancy_sweep.py --counts 8,16,34,64 >> gpurun_out/occ_pdl.txt 2>&1
tail -3 gpurun_out/pytest_q.txt; echo PDL; cat gpurun_out/occ_pdl.txt; echo NOPDL; cat gpurun_out/occ_nopdl.txt

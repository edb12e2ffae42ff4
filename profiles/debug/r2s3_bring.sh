# conv2 forward with a decoupled weight-image B ring (4 / 6 / 8 slots): GPU tests, kernel A/B, lockstep A/B
mkdir -p gpurun_out
V=$PWD/profiles/debug/var
timeout 900 python -m pytest tests/test_cnn_gpu.py tests/test_headline_gpu.py -x -q -p no:cacheprovider --timeout 180 2>&1 | tail -1
timeout 600 python profiles/debug/kbench.py $V/libsmx_BASE.so $V/libsmx_R4.so $V/libsmx_R6.so $V/libsmx_R8.so $V/libsmx_BASE.so $V/libsmx_R6.so
for rep in 1 2; do
  for lib in BASE R6; do
    echo "== $lib"; SMX_LIB_PATH=$V/libsmx_$lib.so timeout 300 python profiles/occupancy_sweep.py --steps 30 --counts 6,12,48,64 | python -c "import sys,json; print(' '.join('%d:%.4f' % (d['slots'], d['ms_per_lockstep']) for d in map(json.loads, sys.stdin)))"
  done
done

# A/B: lockstep time at 8 / 16 / 34 / 64 slots, HEAD worktree (_ab/h) vs this tree, alternated
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_cnn_gpu.py tests/test_headline_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -1
for rep in 1 2; do
  for t in _ab/h .; do
    (cd $t && timeout 300 python profiles/occupancy_sweep.py --counts 8,16,34,64 2>&1 | sed "s|^|$t |")
  done
done

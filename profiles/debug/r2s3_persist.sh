# persistent conv grids: GPU tests, kernel A/B and lockstep-vs-slots A/B against the previous build
mkdir -p gpurun_out
V=$PWD/profiles/debug/var
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 300 2>&1 | tail -2
for rep in 1 2; do
  for lib in NEW7 NEW8; do
    echo "== $lib"; SMX_LIB_PATH=$V/libsmx_$lib.so timeout 300 python profiles/occupancy_sweep.py --steps 30 --counts 6,10,12,34,48,64 | python -c "import sys,json; print(' '.join('%d:%.4f' % (d['slots'], d['ms_per_lockstep']) for d in map(json.loads, sys.stdin)))"
  done
done

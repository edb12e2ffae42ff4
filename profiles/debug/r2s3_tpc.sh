# A/B of the tiles-per-CTA choice: lockstep time vs active slots (C2's counts), alternated
mkdir -p gpurun_out
V=$PWD/profiles/debug/var
for rep in 1 2; do
  for lib in NEW7 T8 T16; do
    echo "== $lib"; SMX_LIB_PATH=$V/libsmx_$lib.so timeout 300 python profiles/occupancy_sweep.py --steps 30 --counts 6,10,12,34,48,64 | python -c "import sys,json; print(' '.join('%d:%.4f' % (d['slots'], d['ms_per_lockstep']) for d in map(json.loads, sys.stdin)))"
  done
done

# A/B of the 64-slot CNN lockstep (CUDA events, profiles/lockstep_probe.py) for library builds,
# alternating 3 times: ab_lockstep.sh lib_a.so lib_b.so ...
for i in 1 2 3; do
  for lib in "$@"; do
    echo -n "$(basename $lib) "; SMX_LIB_PATH=$(realpath $lib) timeout 120 python profiles/lockstep_probe.py --model cnn --slots 64 --steps 10 --warmup 3 --bs 128 2>&1 | tail -1 | sed 's/.*ms\/lockstep/ms\/lockstep/'
  done
done

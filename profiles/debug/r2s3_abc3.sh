# C3 (MLP) bench A/B: round-1 end (_ab/r1), session start (_ab/s0), this tree; alternated twice
mkdir -p gpurun_out
for rep in 1; do
for t in _ab/r1 .; do
  (cd $t && timeout 600 python bench.py --workload c3 --steps 2 --warmup 1 --no-cpu --no-trial 2>/tmp/abc3.err | tail -1) > gpurun_out/abc3.json; tail -3 /tmp/abc3.err
  python -c "
import json; d=json.loads(open('gpurun_out/abc3.json').read()); print('$t', round(d['value']), d['ms_per_step'], d['clocks']['sm_mhz'])"
done
done

# the non-default workloads on one GPU (C3 MLP random search, C4 SHA / ASHA, C5 multi-study)
mkdir -p gpurun_out
for w in c3 c4_sha c4_asha c5; do
  timeout 900 python bench.py --workload $w --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
  echo "$w rc $?"; python -c "
import json; d=json.loads(open('gpurun_out/bench_$w.json').read().strip().splitlines()[-1]); print('$w', round(d['value']), d['unit'], 'e2e', round(d['e2e']['value']), 'savings', d.get('gpu_seconds_savings',{}).get('ratio'))"
done

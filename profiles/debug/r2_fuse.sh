set -x
python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
for m in cnn mlp; do python profiles/lockstep_probe.py --model $m --steps 5 --warmup 2 2>&1 | tail -1; done
for m in cnn mlp; do timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_lockstep_$m.csv python profiles/lockstep_probe.py --model $m --steps 1 --warmup 1 > /dev/null 2>&1; python profiles/launches.py gpurun_out/launches_lockstep_$m.csv 20 > gpurun_out/launches_lockstep_$m.txt; tail -22 gpurun_out/launches_lockstep_$m.txt; done
timeout 900 python bench.py --no-trial > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; python -c "import json;d=json.load(open('gpurun_out/bench_c2.json'));print(d['value'],d['e2e']['value'],d['engine_stats']['locksteps'],d['cpu_baseline']['value'], d['clocks'])"
timeout 900 python bench.py --workload c3 --no-cpu --no-trial > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; python -c "import json;d=json.load(open('gpurun_out/bench_c3.json'));print(d['value'],d['e2e']['value'],d['engine_stats']['locksteps'])"

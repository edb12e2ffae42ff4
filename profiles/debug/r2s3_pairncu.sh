mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.max --clock-control none --kernel-name-base demangled -k "regex:Wgrad" --csv --log-file gpurun_out/pair_ncu.csv python profiles/lockstep_probe.py --model cnn --slots 64 --steps 1 --warmup 1 --max-batch 128 > /dev/null 2>&1
python3 - <<'PY'
import csv
rows=list(csv.reader(open("gpurun_out/pair_ncu.csv")))
h=next(i for i,r in enumerate(rows) if "Kernel Name" in r); hd=rows[h]
for r in rows[h+1:]:
    print(r[hd.index("Kernel Name")][:70], r[hd.index("Grid Size")], r[hd.index("Metric Name")], r[hd.index("Metric Value")])
PY

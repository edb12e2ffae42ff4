# per-kernel elapsed SM cycles (clock-independent) of one 64-slot lockstep, base vs a variant
mkdir -p gpurun_out
for v in base ${1:-nobimg}; do
  if [ $v = base ]; then L=""; else L="SMX_LIB_PATH=profiles/debug/var/libsmx_$v.so"; fi
  env $L timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.max,smsp__cycles_active.avg --clock-control none -k "regex:conv_ws|wgrad|conv1|head|reduce|weight_image" -s 14 -c 14 --csv --log-file gpurun_out/cyc_$v.csv python profiles/lockstep_probe.py --model cnn --slots 64 --steps 2 --warmup 1 > /dev/null 2>&1
  python3 - gpurun_out/cyc_$v.csv $v <<'PY'
import csv,sys,re
rows=list(csv.reader(open(sys.argv[1])))
h=next(i for i,r in enumerate(rows) if 'Kernel Name' in r); hd=rows[h]
ki,mi,vi=hd.index('Kernel Name'),hd.index('Metric Name'),hd.index('Metric Value')
d={}
for r in rows[h+1:]:
    k=re.sub(r'\(.*','',r[ki])[:40]; d.setdefault(k,{})[r[mi]]=float(r[vi].replace(',',''))
for k,m in d.items(): print(sys.argv[2], f"{k:40s} {m.get('gpu__time_duration.sum',0)/1e3:8.1f} us {m.get('sm__cycles_elapsed.max',0)/1e3:8.1f} kcyc  {m.get('sm__cycles_elapsed.max',0)/max(1,m.get('gpu__time_duration.sum',1)):.2f} GHz")
PY
done

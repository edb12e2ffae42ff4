mkdir -p gpurun_out
for v in MMA_NOEPI SKELETON; do
  if [ $v = base ]; then unset SMX_LIB_PATH; else export SMX_LIB_PATH=$PWD/profiles/debug/var/libsmx_$v.so; fi
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/var_$v.csv python profiles/lockstep_probe.py --model cnn --steps 1 --warmup 1 > /dev/null 2>&1
done

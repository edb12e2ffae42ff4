mkdir -p gpurun_out
for k in "regex:conv1_fwd_tc" "regex:conv1_wgrad_tc"; do
  n=$(echo "$k" | tr -dc 'a-zA-Z0-9_')
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "$k" -s 1 -c 1 \
    -o gpurun_out/ncu_$n python profiles/lockstep_probe.py --model cnn --slots 64 --steps 1 --warmup 1 > gpurun_out/ncu_$n.log 2>&1
done
ls -la gpurun_out/*.ncu-rep

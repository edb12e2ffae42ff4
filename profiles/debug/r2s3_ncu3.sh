mkdir -p gpurun_out
for k in "regex:Fwd<\(int\)2>" "regex:Dgrad<\(int\)2>"; do
  n=$(echo "$k" | tr -dc 'a-zA-Z0-9_')
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "$k" -s 1 -c 1 \
    -o gpurun_out/ncu3_$n python profiles/lockstep_probe.py --model cnn --slots 64 --steps 1 --warmup 1 > gpurun_out/ncu3_$n.log 2>&1
done
ls -la gpurun_out/*.ncu-rep

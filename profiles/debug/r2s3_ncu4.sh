mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:head_fwd" -s 1 -c 1 \
    -o gpurun_out/ncu4_head python profiles/lockstep_probe.py --model cnn --slots 64 --steps 1 --warmup 1 > gpurun_out/ncu4.log 2>&1
ls -la gpurun_out/*.ncu-rep

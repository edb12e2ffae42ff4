# one --set full capture of kernel regex $1 from the 64-slot CNN lockstep probe -> gpurun_out/ncu_$2
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$1" -s 0 -c 1 -o gpurun_out/ncu_$2 python profiles/lockstep_probe.py --model cnn --steps 1 --warmup 0 --bs 128 > gpurun_out/ncu_$2.log 2>&1
tail -2 gpurun_out/ncu_$2.log

# bench line + ncu launch list of the bench command (steady state: 2000 launches after the first
# 2000) + one --set full capture of the roofline kernel
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.txt 2> gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 2000 -c 2000 --csv --log-file gpurun_out/bench_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-trial > gpurun_out/bench_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:Wgrad<\(int\)2>" -s 0 -c 1 -o gpurun_out/ncu_wgrad2_full python profiles/lockstep_probe.py --model cnn --steps 1 --warmup 0 --bs 128 > gpurun_out/ncu_full.log 2>&1

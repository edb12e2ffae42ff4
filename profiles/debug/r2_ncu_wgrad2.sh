# one --set full capture of the conv2 weight gradient (64 groups, bs 128) + a lockstep launch list
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:Wgrad<\(int\)2>" -s 0 -c 1 -o gpurun_out/ncu_wgrad2_full python profiles/lockstep_probe.py --model cnn --steps 1 --warmup 0 --bs 128 > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cnn.csv python profiles/lockstep_probe.py --model cnn --steps 2 --warmup 1 --bs 128 > gpurun_out/ncu_ls.log 2>&1
tail -3 gpurun_out/ncu_full.log

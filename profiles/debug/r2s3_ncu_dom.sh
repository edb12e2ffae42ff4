# --set full capture of the bench's roofline kernel (the conv2 input gradient) at the bench
# configuration (64 slots, bs 128, max_batch 128) + the 64-slot lockstep launch list
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:Dgrad<\(int\)2>" -s 1 -c 1 -o gpurun_out/ncu_dgrad2_$1 python profiles/lockstep_probe.py --model cnn --steps 1 --warmup 1 --bs 128 --max-batch 128 > gpurun_out/ncu_dom.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cnn_$1.csv python profiles/lockstep_probe.py --model cnn --steps 2 --warmup 1 --bs 128 --max-batch 128 > /dev/null 2>&1
python profiles/launches.py gpurun_out/launches_cnn_$1.csv 15

# --set full captures of the eight tensor-core conv kernels of one 64-slot CNN lockstep (bs 128,
# max_batch 128 = the bench configuration) + the lockstep launch list, into gpurun_out/
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:Fwd|Dgrad|Wgrad|wgrad2_at|conv1_" -s 0 -c 8 -o gpurun_out/ncu_convs_$1 python profiles/lockstep_probe.py --model cnn --steps 1 --warmup 0 --bs 128 --max-batch 128 > gpurun_out/ncu_convs.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cnn_$1.csv python profiles/lockstep_probe.py --model cnn --steps 2 --warmup 1 --bs 128 --max-batch 128 > gpurun_out/ncu_ls.log 2>&1
tail -2 gpurun_out/ncu_convs.log; python profiles/launches.py gpurun_out/launches_cnn_$1.csv 15

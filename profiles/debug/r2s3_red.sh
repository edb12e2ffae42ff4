# weight-gradient reductions: per-launch times (ncu) of the old / new build in a 64-slot lockstep + GPU tests
mkdir -p gpurun_out
V=$PWD/profiles/debug/var
timeout 600 python -m pytest tests/test_cnn_gpu.py tests/test_headline_gpu.py -x -q -p no:cacheprovider --timeout 180 2>&1 | tail -1
for lib in NEW7 NEW9; do
  SMX_LIB_PATH=$V/libsmx_$lib.so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:wgrad_reduce --csv --log-file gpurun_out/red_$lib.csv python profiles/lockstep_probe.py --model cnn --steps 2 --warmup 1 --bs 128 --max-batch 128 > /dev/null 2>&1
  echo $lib; grep -o '"[^"]*wgrad_reduce[^"]*".*' gpurun_out/red_$lib.csv | awk -F'","' '{print $1, $NF}' | tail -4
done

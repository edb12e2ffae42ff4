# weight images without the never-read rows: GPU tests + per-launch ncu time of weight_image_kernel
mkdir -p gpurun_out
V=$PWD/profiles/debug/var
timeout 600 python -m pytest tests/test_cnn_gpu.py tests/test_headline_gpu.py -x -q -p no:cacheprovider --timeout 180 2>&1 | tail -1
for lib in BASE NEW11 BASE NEW11; do
  SMX_LIB_PATH=$V/libsmx_$lib.so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:weight_image --csv --log-file gpurun_out/wimg_$lib.csv python profiles/lockstep_probe.py --model cnn --steps 2 --warmup 1 --bs 128 --max-batch 128 > /dev/null 2>&1
  echo $lib $(grep -o '"[^"]*weight_image[^"]*".*' gpurun_out/wimg_$lib.csv | awk -F'","' '{print $NF}' | tail -3 | tr '\n' ' ')
done

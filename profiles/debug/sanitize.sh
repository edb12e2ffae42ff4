# compute-sanitizer passes over the smoke path (MLP exact, CNN tensor-core lockstep, Fig. 1 engine
# study) and a 4-slot CNN tensor-core lockstep probe; summaries into gpurun_out/sanitize_*.txt
mkdir -p gpurun_out
for tool in memcheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 \
    python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitize_smoke_$tool.txt 2>&1
  echo "rc $?" >> gpurun_out/sanitize_smoke_$tool.txt
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 \
    python profiles/lockstep_probe.py --model cnn --slots 4 --steps 1 --warmup 1 > gpurun_out/sanitize_cnn_$tool.txt 2>&1
  echo "rc $?" >> gpurun_out/sanitize_cnn_$tool.txt
done
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 --error-exitcode 9 \
  python profiles/lockstep_probe.py --model cnn --slots 2 --steps 1 --warmup 0 > gpurun_out/sanitize_cnn_racecheck.txt 2>&1
echo "rc $?" >> gpurun_out/sanitize_cnn_racecheck.txt
for f in gpurun_out/sanitize_*.txt; do echo "== $f"; tail -4 $f; done

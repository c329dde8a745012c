# GPU box: compute-sanitizer memcheck / synccheck / racecheck of every kernel family (tools/sanitize_smoke.py)
for t in memcheck synccheck racecheck; do
  timeout 1500 compute-sanitizer --tool $t python tools/sanitize_smoke.py > gpurun_out/sanitizer_$t.log 2>&1
  echo "$t rc=$?"; tail -2 gpurun_out/sanitizer_$t.log
done

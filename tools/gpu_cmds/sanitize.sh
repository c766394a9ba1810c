timeout 600 python tools/sanitize_smoke.py || exit 1
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_smoke.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "== $tool rc=$?"; tail -3 gpurun_out/sanitize_$tool.log
done

# compute-sanitizer over every device code path (tools/sanitize_run.py), one tool per run.
# usage (GPU box): bash tools/sanitize.sh  -> gpurun_out/sanitize_<tool>.txt
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 \
    python tools/sanitize_run.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitize_$tool.txt
done

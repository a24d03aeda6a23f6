# compute-sanitizer evidence: memcheck, racecheck, synccheck, initcheck over
# tools/sanitize.py's cases; logs in gpurun_out/sanitize_<tool>.log
o=gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 \
    python tools/sanitize.py fwd bf16 window host wide simt > $o/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" | tee -a $o/sanitize_summary.txt
  tail -3 $o/sanitize_$tool.log
done

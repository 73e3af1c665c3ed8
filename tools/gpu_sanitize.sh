mkdir -p gpurun_out
timeout 600 python tools/sanitize_paths.py > gpurun_out/sanitize_plain.txt 2>&1; echo "plain rc=$?"; tail -2 gpurun_out/sanitize_plain.txt
for tool in memcheck synccheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_paths.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|all paths ok|Error" gpurun_out/sanitize_$tool.txt | head -5
done

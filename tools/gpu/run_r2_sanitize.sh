# round 2: compute-sanitizer memcheck / racecheck / synccheck on one cfg1-bf16 mixed iteration, temporal and spatial
mkdir -p gpurun_out
for tool in memcheck synccheck racecheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_step.py --config cfg1-bf16 \
    > gpurun_out/sanitize_$tool.log 2>&1
  echo "== $tool rc=$?"; grep -E "ERROR SUMMARY|sanitize cfg1|Error|error" gpurun_out/sanitize_$tool.log | head -8
done

# round 2: sanitizers on cfg2-mini (tcgen05 attention kernels, d_h = 128), trace with burst calibration
mkdir -p gpurun_out
for tool in memcheck synccheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_step.py --config cfg2-mini \
    > gpurun_out/sanitize2_$tool.log 2>&1
  echo "== $tool rc=$?"; grep -E "ERROR SUMMARY|sanitize cfg2" gpurun_out/sanitize2_$tool.log | head -4
  grep "Race reported" gpurun_out/sanitize2_$tool.log | sed 's/.*at void //; s/(CUtensor.*//; s/+0x.*//' | sort | uniq -c | head
done
timeout 2400 python tools/trace_bench.py --n-req 48 --qps 40 --max-iters 8000 --calibration burst --out gpurun_out/trace_cfg4_burst.json > gpurun_out/trace_burst.log 2>&1
grep -E "^(static|static_slo|adaptive) " gpurun_out/trace_burst.log | cut -c1-330

mkdir -p gpurun_out
DUET_FA_TRACE=1 timeout 300 python bench.py --profile-only --steps 1 --warmup 1 --no-cpu-baseline 2>/dev/null | grep FA_TRACE | head -40 > gpurun_out/fa_trace.txt
cat gpurun_out/fa_trace.txt
